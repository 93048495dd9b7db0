"""Seeded randomised parity sweep: random supported shapes, appends in random
chunk sizes (odd counts, pairs split across calls), random sink tokens,
ragged decode lengths, both scale formats and (a quarter of the cases) the
fused-frame append of the oracle's rotated + reordered fp32 rows
(rkv_quantize_kv_fused).  Every case checks the cache
bit for bit against the oracle (codes, scale|zero words, sink rows, mask)
and decode (and, on the tensor-core shapes, prefill) against the oracle's
attention at the bar of test_gpu_parity.py.  Deterministic: case i uses
numpy seed 1000 + i.  RKV_FUZZ_CASES widens the sweep (default 85)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

from .test_gpu_parity import (COS_TOL, REL_TOL, build_layer, cache_host, cosine, oracle_decode,  # noqa: E402
                             rel_err, small_workload)

# (Hq, Hkv, G): tensor-core MHA at G = 1/2/4 (up to C = 8192), GQA (any ratio) at G = 2
# and 4, CUDA-core shapes, generic (tiled) shapes
SHAPES = [(8, 8, 4), (8, 8, 2), (8, 8, 1), (12, 12, 4), (40, 40, 4), (16, 4, 2), (32, 8, 2), (16, 8, 4),
          (8, 4, 2), (16, 4, 1), (4, 4, 1), (16, 4, 4), (32, 8, 4), (64, 64, 4), (16, 16, 8), (24, 8, 8),
          (64, 16, 4), (64, 8, 2), (32, 4, 4), (40, 8, 2), (24, 8, 4), (16, 8, 2)]
TC_PREFILL = {(8, 8, 4), (8, 8, 2), (8, 8, 1), (12, 12, 4), (40, 40, 4), (16, 4, 2), (32, 8, 2), (4, 4, 1),
              (16, 8, 4), (8, 4, 2),
              (16, 4, 4), (32, 8, 4), (64, 64, 4), (64, 8, 2), (32, 4, 4), (40, 8, 2), (24, 8, 4), (16, 8, 2)}


def case(i):
    rng = np.random.default_rng(1000 + i)
    hq, hkv, g = SHAPES[i % len(SHAPES)]
    B = int(rng.integers(1, 4))
    T = int(rng.integers(2, 330))
    fmt = P.SCALE_E4M3_CEIL if rng.random() < 0.3 else P.SCALE_FP16_CEIL
    chunks = []
    left = T
    while left:
        n = int(min(left, rng.integers(1, 97)))
        chunks.append(n)
        left -= n
    flags = (rng.random((B, T)) < 0.01).astype(np.uint8)
    flags[:, 0] = 1
    lens = [int(rng.integers(1, T + 1)) for _ in range(B)]
    lens[int(rng.integers(0, B))] = T
    base = 500000.0 if rng.random() < 0.5 else 10000.0
    return dict(hq=hq, hkv=hkv, g=g, B=B, T=T, fmt=fmt, chunks=chunks, flags=flags, lens=lens, base=base,
                fused=bool(rng.random() < 0.25))


@pytest.mark.parametrize("i", range(int(os.environ.get("RKV_FUZZ_CASES", "85"))))  # wider sweeps: RKV_FUZZ_CASES=400
def test_random_case(oracle, i):
    c = case(i)
    w = small_workload(c["hq"], c["hkv"], c["g"], base=c["base"])
    B, T = c["B"], c["T"]
    max_sinks = int(c["flags"].sum(axis=1).max()) + 1
    layer, perm = build_layer(w, B, T + 3, seed=1000 + i, fmt=c["fmt"], max_sinks=max_sinks)
    k, v = WL.make_kv(w, 1000 + i, B, T)
    flags = torch.from_numpy(c["flags"])
    if c["fused"]:  # K' = reorder(H_G k), V' = H_128 v in fp32 (the reference's fused projections)
        C = w.channels
        kf = oracle.apply_reorder(oracle.rotate_rows(k.float().cpu().numpy().reshape(-1, C), 128, c["g"], c["hkv"]), perm)
        vf = oracle.rotate_rows(v.float().cpu().numpy().reshape(-1, C), 128, 1, c["hkv"])
        kf = torch.from_numpy(kf.reshape(B, T, C)).cuda()
        vf = torch.from_numpy(vf.reshape(B, T, C)).cuda()
    t0 = 0
    for n in c["chunks"]:
        if c["fused"]:
            layer.append_fused(kf[:, t0:t0 + n], vf[:, t0:t0 + n], flags[:, t0:t0 + n])
        else:
            layer.append(k[:, t0:t0 + n], v[:, t0:t0 + n], flags[:, t0:t0 + n])
        t0 += n
    torch.cuda.synchronize()
    got = cache_host(layer)
    kh, vh = k.cpu().numpy(), v.cpu().numpy()
    for b in range(B):
        kc, km, vc, vm = oracle.quantize_kv_rows(kh[b], vh[b], c["hkv"], 128, c["g"], perm, c["fmt"])
        s = c["flags"][b].astype(bool)
        for a in (kc, km, vc, vm):
            a[s] = 0
        assert np.array_equal(got["k_codes"][b, :T].view(np.uint32), kc), (i, b)
        assert np.array_equal(got["k_meta"][b, :T].view(np.uint32), km), (i, b)
        assert np.array_equal(got["v_codes"][b, :T].view(np.uint32), vc), (i, b)
        assert np.array_equal(got["v_meta"][b, :T].view(np.uint32), vm), (i, b)
        pos = np.flatnonzero(s)
        assert got["sink_count"][b] == len(pos)
        assert list(got["sink_pos"][b, :len(pos)]) == list(pos)
        for j, t in enumerate(pos):
            if not c["fused"]:
                assert np.array_equal(got["sink_k"][b, j].view(np.uint16), kh[b, t].view(np.uint16))
            else:  # back through the inverse reorder and FWHT: within an fp16 rounding
                x = kh[b, t].astype(np.float32)
                y = got["sink_k"][b, j].view(np.float16).astype(np.float32)
                assert np.all(np.abs(x - y) <= 1e-3 * np.abs(x) + 1e-5 * np.max(np.abs(x))), (i, b, t)
    q = WL.make_q(w, 1000 + i, B)
    out = layer.decode(q, seq_len=c["lens"]).cpu().numpy()
    for b, L in enumerate(c["lens"]):
        want = oracle_decode(oracle, layer, got, b, L, q[b].cpu().numpy(), w, perm, kh[b], vh[b])
        assert rel_err(out[b], want) < REL_TOL, (i, b, L)
        assert cosine(out[b], want) > COS_TOL, (i, b, L)
    if (c["hq"], c["hkv"], c["g"]) in TC_PREFILL and max_sinks <= 16:
        # the last rows of the full-length sequence's prompt, queries at their own positions
        nq = min(T, 24)
        qs = WL.make_q(w, 2000 + i, B * nq).reshape(B, nq, c["hq"], 128)
        start = np.full(B, T - nq, np.int64)
        pre = layer.prefill_attention(qs, q_start=start).cpu().numpy()
        b = int(np.argmax(c["lens"]))
        for r in (0, nq // 2, nq - 1):
            want = oracle_decode(oracle, layer, got, b, T - nq + r + 1, qs[b, r].cpu().numpy(), w, perm, kh[b], vh[b])
            assert rel_err(pre[b, r], want) < REL_TOL, (i, r)
