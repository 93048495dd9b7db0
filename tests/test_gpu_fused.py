"""Fused-frame append (rkv_quantize_kv_fused).

With fuse_weights (proj/src/pipeline.cpp:88-99) the reference's projections
emit K' = P H_G k and V' = H_128 v and LayerKVCache::append
(proj/src/kv_cache.cpp:8-22) only quantizes them.  These tests feed the
oracle's K' / V' (rotate_rows + apply_reorder in fp32, the on-the-fly chain's
own intermediate) to the fused path and require the cache to equal the
on-the-fly path's for the raw rows: packed words and metadata bit-exact,
sink rows back in the model frame, decode within the north-star bar.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

from tests.test_gpu_parity import (COS_TOL, REL_TOL, build_layer, cache_host, cosine, oracle_decode,  # noqa: E402
                             rel_err, small_workload)

PACKED = ("k_codes", "k_meta", "v_codes", "v_meta")


def same_cache(ga, gf, T):
    """Written rows [0, T) of the packed arrays, the sink masks, counts and
    used sidecar slots equal (sidecar rows: K' / V' back through the inverse
    reorder and FWHT, rounded to fp16 -- within an fp16 rounding)."""
    for name in PACKED:
        assert np.array_equal(ga[name][:, :T], gf[name][:, :T]), name
    for name in ("sink_mask", "sink_count"):
        assert np.array_equal(ga[name], gf[name]), name
    for b, n in enumerate(ga["sink_count"]):
        assert np.array_equal(ga["sink_pos"][b, :n], gf["sink_pos"][b, :n])
        for name in ("sink_k", "sink_v"):
            x = ga[name][b, :n].view(np.float16).astype(np.float32)
            y = gf[name][b, :n].view(np.float16).astype(np.float32)
            # one fp16 rounding of an fp32 value within ~1e-6 of the original
            tol = 1e-3 * np.abs(x) + 1e-5 * np.max(np.abs(x), axis=-1, keepdims=True)
            assert np.all(np.abs(x - y) <= tol), (name, float(np.max(np.abs(x - y))))


def fused_rows(oracle, w, perm, k, v):
    """K' = apply_reorder(rotate_rows(k, G)), V' = rotate_rows(v, 1): fp32 [B, T, C]."""
    B, T, C = k.shape
    kf = oracle.rotate_rows(k.float().cpu().numpy().reshape(-1, C), 128, w.heads_per_group, w.num_kv_heads)
    kf = oracle.apply_reorder(kf, perm)
    vf = oracle.rotate_rows(v.float().cpu().numpy().reshape(-1, C), 128, 1, w.num_kv_heads)
    return (torch.from_numpy(kf.reshape(B, T, C)).cuda(), torch.from_numpy(vf.reshape(B, T, C)).cuda())


@pytest.mark.parametrize("hq,hkv,g,fmt,T", [
    (8, 8, 4, P.SCALE_FP16_CEIL, 37), (40, 40, 4, P.SCALE_FP16_CEIL, 64), (32, 8, 2, P.SCALE_FP16_CEIL, 33),
    (8, 8, 4, P.SCALE_E4M3_CEIL, 20), (4, 4, 1, P.SCALE_FP16_CEIL, 9),
    # C = 512 and 1536: the last 1024-slot segment is partly idle
    (16, 4, 1, P.SCALE_FP16_CEIL, 17), (12, 12, 4, P.SCALE_FP16_CEIL, 15),
    (64, 64, 8, P.SCALE_FP16_CEIL, 7),  # C = 8192, n = 1024 (the generic on-the-fly kernel)
])
def test_fused_append_equals_on_the_fly(oracle, hq, hkv, g, fmt, T):
    w = small_workload(hq, hkv, g)
    B = 2
    a, perm = build_layer(w, B, T + 8, seed=T + g, fmt=fmt)
    f, _ = build_layer(w, B, T + 8, seed=T + g, fmt=fmt, perm=perm)
    k, v = WL.make_kv(w, T + g, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    sinks[1, T // 2] = 1
    a.append(k, v, sinks)
    kf, vf = fused_rows(oracle, w, perm, k, v)
    f.append_fused(kf, vf, sinks)
    torch.cuda.synchronize()
    ga, gf = cache_host(a), cache_host(f)
    same_cache(ga, gf, T)
    q = WL.make_q(w, T, B)
    oa, of = a.decode(q).cpu().numpy(), f.decode(q).cpu().numpy()
    assert rel_err(of, oa) < 1e-3
    for b in range(B):
        want = oracle_decode(oracle, f, gf, b, T, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(of[b], want) < REL_TOL
        assert cosine(of[b], want) > COS_TOL


@pytest.mark.parametrize("hq,hkv,g", [(8, 8, 4), (32, 8, 2)])
def test_fused_fp16_rows_equal_fp32_rows_of_the_same_values(hq, hkv, g):
    """RKV_ROWS_F16 quantizes the fp16 values exactly as RKV_ROWS_F32 does their fp32 image."""
    w = small_workload(hq, hkv, g)
    B, T = 2, 45
    a, perm = build_layer(w, B, T, seed=9)
    f, _ = build_layer(w, B, T, seed=9, perm=perm)
    gen = torch.Generator().manual_seed(9)
    k16 = (torch.randn(B, T, w.channels, generator=gen) * 3).half().cuda()
    v16 = torch.randn(B, T, w.channels, generator=gen).half().cuda()
    a.append_fused(k16.float(), v16.float())
    f.append_fused(k16, v16)
    torch.cuda.synchronize()
    ga, gf = cache_host(a), cache_host(f)
    same_cache(ga, gf, T)


def test_fused_append_matches_unmodified_reference_e4m3(ref):
    """e4m3 scales: the words equal the unmodified reference's rotate -> reorder
    -> quantize_token chain on the raw rows (proj/src/pipeline.cpp:317-324)."""
    w = small_workload(8, 8, 4)
    B, T = 1, 24
    f, perm = build_layer(w, B, 32, seed=3, fmt=P.SCALE_E4M3_CEIL)
    k, v = WL.make_kv(w, 3, B, T)
    kr = ref.rotate_rows(k[0].float().cpu().numpy(), 128, 4, 8, impl="ref")
    kr = ref.apply_reorder(kr, perm, impl="ref")
    vr = ref.rotate_rows(v[0].float().cpu().numpy(), 128, 1, 8, impl="ref")
    f.append_fused(torch.from_numpy(kr).reshape(1, T, -1).cuda(), torch.from_numpy(vr).reshape(1, T, -1).cuda())
    torch.cuda.synchronize()
    got = cache_host(f)
    kc, ks, kz, vc, vs, vz = ref.ref_quantize_kv_rows(k[0].float().cpu().numpy(), v[0].float().cpu().numpy(),
                                                     8, 128, 4, perm)
    assert np.array_equal(got["k_codes"][0, :T].view(np.uint32), kc)
    assert np.array_equal(got["v_codes"][0, :T].view(np.uint32), vc)
    dec = np.vectorize(lambda c: ref.e4m3_decode(int(c)))
    km = got["k_meta"][0, :T].view(np.uint32)
    assert np.array_equal((km & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float32), dec(ks))
    assert np.array_equal((km >> 16).astype(np.uint16).view(np.float16).astype(np.float32), kz.astype(np.float32))
    vm = got["v_meta"][0, :T].view(np.uint32)
    assert np.array_equal((vm & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float32), dec(vs))


def test_fused_odd_counts_offsets_and_sinks(oracle):
    """Odd token counts (a pair's second token absent), appends at an offset
    and several sinks per call, as the on-the-fly path does."""
    w = small_workload(16, 16, 4)
    B = 3
    a, perm = build_layer(w, B, 64, seed=21, max_sinks=2)
    f, _ = build_layer(w, B, 64, seed=21, perm=perm, max_sinks=2)
    for step, n in enumerate((5, 1, 12)):
        k, v = WL.make_kv(w, 30 + step, B, n)
        flags = torch.zeros(B, n, dtype=torch.uint8)
        if step == 0:
            flags[:, 0] = 1
            flags[2, 3] = 1  # sequence 2 fills its two-slot sidecar
        a.append(k, v, flags)
        kf, vf = fused_rows(oracle, w, perm, k, v)
        f.append_fused(kf, vf, flags)
    torch.cuda.synchronize()
    ga, gf = cache_host(a), cache_host(f)
    same_cache(ga, gf, 18)
    assert list(gf["sink_count"]) == [1, 1, 2]


def test_fused_errors():
    w = small_workload(8, 8, 4)
    f, _ = build_layer(w, 1, 16, seed=1)
    k = torch.zeros(1, 4, w.channels, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        f.append_fused(k, k)
    k = torch.zeros(1, 4, w.channels + 128, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        f.append_fused(k, k)
    k = torch.zeros(1, 20, w.channels, dtype=torch.float32, device="cuda")
    with pytest.raises(IndexError):
        f.append_fused(k, k)
