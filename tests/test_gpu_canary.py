"""Out-of-bounds write canaries for every kernel family.

compute-sanitizer is not available on the GPU pool, so the bounds are checked
from the outside: the carved cache, the decode / prefill outputs and their
workspaces each sit between 64 KiB guard bands filled with a byte pattern,
the entry points run at shapes that put the last rows of the cache, the last
sequence and the last mask word in play (max_tokens not a multiple of 32, a
full cache, a full sink sidecar, ragged decode lengths), and afterwards every guard
byte must be unchanged.  The guarded runs must also give bit-identical
results to the same calls on ordinary allocations (the kernels are
deterministic).
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import rotatekv as RK  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

from tests.test_gpu_parity import build_layer, small_workload  # noqa: E402

PAD = 65536
PAT = 0xA5


class Guarded:
    """nbytes of device memory at a 64 KiB-aligned offset inside a buffer whose
    remaining bytes hold PAT."""

    def __init__(self, nbytes):
        self.n = max(int(nbytes), 1)
        self.buf = torch.full((PAD + self.n + PAD,), PAT, dtype=torch.uint8, device="cuda")
        self.ptr = self.buf.data_ptr() + PAD

    def view(self, dtype, shape):
        esz = torch.empty((), dtype=dtype).element_size()
        return self.buf[PAD:PAD + int(np.prod(shape)) * esz].view(dtype).view(*shape)

    def check(self, what):
        torch.cuda.synchronize()
        lo, hi = self.buf[:PAD], self.buf[PAD + self.n:]
        bad_lo = int((lo != PAT).sum())
        bad_hi = int((hi != PAT).sum())
        assert bad_lo == 0 and bad_hi == 0, f"{what}: {bad_lo} guard bytes before / {bad_hi} after overwritten"


def guard_cache(layer):
    """Re-carve the layer's cache inside guard bands (then reset it)."""
    nbytes = RK.lib().rkv_cache_bytes(C.byref(layer._desc))
    g = Guarded(nbytes)
    RK._check(RK.lib().rkv_cache_carve(C.byref(layer._desc), g.ptr, nbytes, C.byref(layer._view)))
    layer._buf, layer._base = g.buf, g.ptr
    layer.reset()
    return g


def guarded_decode(layer, q, lens=None):
    B, Hq = layer.cfg.batch, layer.cfg.num_q_heads
    lens = layer.lengths.copy() if lens is None else np.asarray(lens, np.int64)
    msl = int(lens.max())
    need = RK.lib().rkv_decode_workspace_bytes(C.byref(layer._desc), msl)
    ws, out = Guarded(need), Guarded(B * Hq * 128 * 4)
    lens = torch.from_numpy(lens).to("cuda")
    RK._check(RK.lib().rkv_decode_attention(C.byref(layer._desc), RK._ptr(q.contiguous()), RK._ptr(lens), msl,
                                            C.byref(layer._view), RK._ptr(layer.plan), RK._ptr(layer.rope), out.ptr,
                                            ws.ptr, need, layer._stream()))
    ws.check("decode workspace")
    out.check("decode output")
    return out.view(torch.float32, (B, Hq, 128)).clone()


def guarded_prefill(layer, q):
    B, nq, Hq = q.shape[0], q.shape[1], q.shape[2]
    mx = int(layer.lengths.max())
    need = RK.lib().rkv_prefill_workspace_bytes(C.byref(layer._desc), nq, mx)
    ws, out = Guarded(need), Guarded(B * nq * Hq * 128 * 4)
    st = torch.from_numpy(layer.lengths - nq).to("cuda")
    ln = torch.from_numpy(layer.lengths.copy()).to("cuda")
    RK._check(RK.lib().rkv_prefill_attention(C.byref(layer._desc), RK._ptr(q.contiguous()), nq, RK._ptr(st),
                                             RK._ptr(ln), mx, C.byref(layer._view), RK._ptr(layer.plan),
                                             RK._ptr(layer.rope), out.ptr, ws.ptr, need, layer._stream()))
    ws.check("prefill workspace")
    out.check("prefill output")
    return out.view(torch.float32, (B, nq, Hq, 128)).clone()


def assert_same_cache(a, b):
    """Every cache array equal -- the code / metadata rows up to each
    sequence's length and the sidecars in their used slots (reset leaves
    unwritten rows and slots as they were)."""
    ta, tb = a.arrays(), b.arrays()
    counts = ta["sink_count"].cpu().tolist()
    for name, t in ta.items():
        if name in ("k_codes", "v_codes", "k_meta", "v_meta"):
            for s, n in enumerate(a.lengths.tolist()):
                assert torch.equal(t[s, :n], tb[name][s, :n]), f"{name} differs from the unguarded run"
        elif name in ("sink_k", "sink_v", "sink_pos"):
            for s, n in enumerate(counts):
                assert torch.equal(t[s, :n], tb[name][s, :n]), f"{name} differs from the unguarded run"
        else:
            assert torch.equal(t, tb[name]), f"cache array {name} differs from the unguarded run"


# (hq, hkv, G, batch, max_tokens, appended): MHA at G = 4 / 2 / 1, GQA 4:1 at G = 2
# and 4, GQA 8:1 (two head sets), a G = 8 layer (tiled generic kernels), a
# C = 5120 layer with enough token pairs for the warp-independent V kernel, and
# C = 8192 (256 regions per token); max_tokens off the 32-token mask words
CASES = [
    (8, 8, 4, 8, 451, 451),
    (8, 8, 2, 3, 97, 90),
    (8, 8, 1, 2, 70, 70),
    (16, 4, 2, 3, 333, 333),
    (16, 4, 4, 3, 333, 301),
    (64, 8, 2, 2, 129, 129),
    (16, 16, 8, 2, 161, 161),
    (40, 40, 4, 4, 201, 201),
    (64, 64, 4, 2, 65, 65),
]


@pytest.mark.parametrize("hq,hkv,g,B,T,n", CASES)
def test_guard_bands_intact(hq, hkv, g, B, T, n):
    w = small_workload(hq, hkv, g)
    plain, perm = build_layer(w, B, T, seed=93, max_sinks=2)
    guarded, _ = build_layer(w, B, T, seed=93, max_sinks=2, perm=perm)
    gc = guard_cache(guarded)
    k, v = WL.make_kv(w, 93, B, n)
    flags = torch.zeros(B, n, dtype=torch.uint8)
    flags[:, 0] = 1
    flags[B - 1, n - 1] = 1  # a sink in the last row of the last sequence
    for lay in (plain, guarded):
        lay.append(k, v, flags)
    gc.check("quantize_kv")
    assert_same_cache(plain, guarded)

    q = WL.make_q(w, 93, B)
    want = plain.decode(q)
    got = guarded_decode(guarded, q)
    gc.check("decode (cache)")
    assert torch.equal(got, want)
    assert bool(torch.isfinite(got).all())
    ragged = np.maximum(1, n - 37 * np.arange(B, dtype=np.int64))  # ragged lengths: other last tiles and splits
    want = plain.decode(q, seq_len=ragged)
    got = guarded_decode(guarded, q, ragged)
    gc.check("decode, ragged lengths (cache)")
    assert torch.equal(got, want)

    if g == 8:  # prefill: G = 1, 2, 4 only (host-side refusal)
        return
    nq = min(64, n)
    qp = torch.randn(B, nq, hq, 128, generator=torch.Generator().manual_seed(5)).half().cuda()
    wantp = plain.prefill_attention(qp)
    gotp = guarded_prefill(guarded, qp)
    gc.check("prefill (cache)")
    assert torch.equal(gotp, wantp)


@pytest.mark.parametrize("hq,hkv,g", [(8, 8, 4), (40, 40, 4), (16, 4, 2)])
def test_guard_bands_fused_append_and_promote(hq, hkv, g):
    """The fused-frame append (fp32 and fp16 rows, sinks in the first and
    last rows) and post-hoc sink promotion write only inside the cache."""
    w = small_workload(hq, hkv, g)
    B, T = 3, 99
    layer, perm = build_layer(w, B, T, seed=17, max_sinks=2)
    gc = guard_cache(layer)
    C_ = layer.cfg.channels
    rows = torch.randn(B, T, C_, generator=torch.Generator().manual_seed(3)).cuda()
    flags = torch.zeros(B, T, dtype=torch.uint8)
    flags[:, 0] = 1
    flags[:, T - 1] = 1  # the sidecar (2) full after the last row
    layer.append_fused(rows[:, :50], rows[:, :50] * 0.5, flags[:, :50])
    layer.append_fused(rows[:, 50:].half(), (rows[:, 50:] * 0.5).half(), flags[:, 50:])
    gc.check("quantize_kv_fused")
    layer2, _ = build_layer(w, B, T, seed=17, max_sinks=4, perm=perm)
    gc2 = guard_cache(layer2)
    k, v = WL.make_kv(w, 17, B, T)
    layer2.append(k, v)
    toks = np.array([[T - 1, 5], [0, T - 2], [7, -1]], dtype=np.int64)
    kr = torch.stack([k[b, [max(int(t), 0) for t in toks[b]]] for b in range(B)]).cuda()
    vr = torch.stack([v[b, [max(int(t), 0) for t in toks[b]]] for b in range(B)]).cuda()
    layer2.promote_sinks(toks, kr, vr)
    gc2.check("promote_sinks")
