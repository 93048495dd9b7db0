"""GPU parity: the sm_100a kernels through the C ABI vs the CPU oracle
(oracle/rkv_oracle.c) and, where oracle/_ref was built, the unmodified
reference.  Bars (BASELINE.json north_star):
  * packed 2-bit codes, scales and zeros: bit-exact;
  * decode output: max|a-b|/max|b| <= 2e-3 (the reference's rel_diff,
    proj/tests/test_pipeline.cpp:23-27) and cosine >= 0.9999.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

REL_TOL = 2e-3
COS_TOL = 0.9999


def rel_err(a, b):
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-12))


def cosine(a, b):
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    return float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b)))


def small_workload(hq, hkv, g, base=10000.0, outliers=4, gain=(10.0, 30.0)):
    return WL.Workload("test", 1, hq, hkv, 0, g, base, outliers, gain)


def build_layer(w, batch, max_tokens, seed, fmt=P.SCALE_FP16_CEIL, max_sinks=8, perm=None):
    if perm is None:
        perm = WL.calibration_perm(w, seed)
    cfg = P.LayerConfig(batch=batch, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                        heads_per_group=w.heads_per_group, max_tokens=max_tokens, max_sinks=max_sinks,
                        rope_base=w.rope_base, scale_format=fmt)
    return P.RotateKVLayer(cfg, perm), perm


def cache_host(layer):
    a = layer.arrays()
    return {k: v.cpu().numpy() for k, v in a.items()}


# ------------------------------------------------------------- quantize_kv

@pytest.mark.parametrize("hq,hkv,g,fmt", [
    (8, 8, 4, P.SCALE_FP16_CEIL), (8, 8, 2, P.SCALE_FP16_CEIL), (4, 4, 1, P.SCALE_FP16_CEIL),
    (40, 40, 4, P.SCALE_FP16_CEIL), (32, 8, 2, P.SCALE_FP16_CEIL), (8, 8, 4, P.SCALE_E4M3_CEIL),
    (40, 40, 4, P.SCALE_E4M3_CEIL),
    # the widest rows (C = 8192; 256 regions per token) and a narrow 4:1 GQA layer at G = 1 (C = 512)
    (64, 64, 4, P.SCALE_FP16_CEIL), (64, 64, 1, P.SCALE_E4M3_CEIL), (16, 4, 1, P.SCALE_FP16_CEIL),
])
def test_quantize_kv_bit_exact_vs_oracle(oracle, hq, hkv, g, fmt):
    w = small_workload(hq, hkv, g)
    B, T = 2, 37
    layer, perm = build_layer(w, B, 64, seed=1, fmt=fmt)
    k, v = WL.make_kv(w, 1, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    sinks[1, 20] = 1
    layer.append(k, v, sinks)
    torch.cuda.synchronize()
    got = cache_host(layer)
    kh = k.cpu().numpy()
    vh = v.cpu().numpy()
    for b in range(B):
        kc, km, vc, vm = oracle.quantize_kv_rows(kh[b], vh[b], hkv, 128, g, perm, fmt)
        s = sinks[b].numpy().astype(bool)
        kc[s] = 0
        km[s] = 0
        vc[s] = 0
        vm[s] = 0
        assert np.array_equal(got["k_codes"][b, :T].view(np.uint32), kc)
        assert np.array_equal(got["k_meta"][b, :T].view(np.uint32), km)
        assert np.array_equal(got["v_codes"][b, :T].view(np.uint32), vc)
        assert np.array_equal(got["v_meta"][b, :T].view(np.uint32), vm)
        pos = np.flatnonzero(s)
        assert got["sink_count"][b] == len(pos)
        assert list(got["sink_pos"][b, :len(pos)]) == list(pos)
        for i, t in enumerate(pos):
            assert np.array_equal(got["sink_k"][b, i].view(np.uint16), kh[b, t].view(np.uint16))
            assert np.array_equal(got["sink_v"][b, i].view(np.uint16), vh[b, t].view(np.uint16))
        mask = got["sink_mask"][b].view(np.uint32)
        bits = [(mask[t // 32] >> (t % 32)) & 1 for t in range(T)]
        assert bits == list(s.astype(int))


def test_quantize_kv_e4m3_matches_unmodified_reference(ref):
    """E4M3 mode vs the reference's own rotate_rows -> apply_reorder ->
    quantize_token (compiled from /root/reference, oracle/_ref)."""
    w = small_workload(8, 8, 4)
    B, T = 1, 48
    layer, perm = build_layer(w, B, 64, seed=3, fmt=P.SCALE_E4M3_CEIL)
    k, v = WL.make_kv(w, 3, B, T)
    layer.append(k, v)
    torch.cuda.synchronize()
    got = cache_host(layer)
    kc, ks, kz, vc, vs, vz = ref.ref_quantize_kv_rows(k[0].float().cpu().numpy(), v[0].float().cpu().numpy(),
                                                     8, 128, 4, perm)
    assert np.array_equal(got["k_codes"][0, :T].view(np.uint32), kc)
    assert np.array_equal(got["v_codes"][0, :T].view(np.uint32), vc)
    dec = np.vectorize(lambda c: ref.e4m3_decode(int(c)))
    km = got["k_meta"][0, :T].view(np.uint32)
    assert np.array_equal((km & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float32), dec(ks))
    assert np.array_equal((km >> 16).astype(np.uint16).view(np.float16).astype(np.float32), kz.astype(np.float32))


def test_quantize_kv_boundary_values_bit_exact(oracle):
    """Rows whose rotated values sit on rounding boundaries: inject rows made
    of a few distinct values so FWHT outputs hit (m-0.5)*s ties."""
    w = small_workload(8, 8, 4)
    B, T = 1, 32
    layer, perm = build_layer(w, B, 32, seed=5)
    rng = np.random.default_rng(5)
    k = rng.integers(-3, 4, size=(B, T, w.channels)).astype(np.float16)
    v = (rng.integers(-2, 3, size=(B, T, w.channels)) * 0.5).astype(np.float16)
    kt = torch.from_numpy(k).cuda()
    vt = torch.from_numpy(v).cuda()
    layer.append(kt, vt)
    torch.cuda.synchronize()
    got = cache_host(layer)
    kc, km, vc, vm = oracle.quantize_kv_rows(k[0], v[0], 8, 128, 4, perm)
    assert np.array_equal(got["k_codes"][0, :T].view(np.uint32), kc)
    assert np.array_equal(got["v_codes"][0, :T].view(np.uint32), vc)
    assert np.array_equal(got["k_meta"][0, :T].view(np.uint32), km)
    assert np.array_equal(got["v_meta"][0, :T].view(np.uint32), vm)


def test_quantize_odd_token_count_and_offsets(oracle):
    """Appends of 1 token at a time and odd counts land at the right rows."""
    w = small_workload(8, 8, 4)
    B = 3
    layer, perm = build_layer(w, B, 40, seed=6)
    k, v = WL.make_kv(w, 6, B, 9)
    layer.append(k[:, :5], v[:, :5])
    for t in range(5, 9):
        layer.append(k[:, t:t + 1], v[:, t:t + 1])
    torch.cuda.synchronize()
    got = cache_host(layer)
    for b in range(B):
        kc, km, vc, vm = oracle.quantize_kv_rows(k[b].cpu().numpy(), v[b].cpu().numpy(), 8, 128, 4, perm)
        assert np.array_equal(got["k_codes"][b, :9].view(np.uint32), kc)
        assert np.array_equal(got["v_meta"][b, :9].view(np.uint32), vm)


# --------------------------------------------------------- decode_attention

def oracle_decode(oracle, layer, got, b, T, q, w, perm, kraw, vraw):
    s = np.zeros(T, np.uint8)
    mask = got["sink_mask"][b].view(np.uint32)
    for t in range(T):
        s[t] = (mask[t // 32] >> (t % 32)) & 1
    return oracle.decode_attention(got["k_codes"][b, :T].view(np.uint32), got["k_meta"][b, :T].view(np.uint32),
                                   got["v_codes"][b, :T].view(np.uint32), got["v_meta"][b, :T].view(np.uint32),
                                   s, kraw[:T], vraw[:T], q, w.num_q_heads, w.num_kv_heads, 128,
                                   w.heads_per_group, perm, w.rope_base)


@pytest.mark.parametrize("hq,hkv,g,base,T", [
    (8, 8, 4, 10000.0, 37), (8, 8, 4, 10000.0, 1), (8, 8, 2, 10000.0, 300),
    (32, 8, 2, 500000.0, 129), (4, 4, 1, 10000.0, 64), (40, 40, 4, 10000.0, 200),
    (16, 8, 4, 10000.0, 77), (32, 32, 4, 10000.0, 1500),
    # per-head (G = 1) and two-head (G = 2) rotations on the 512-channel tensor-core tiles
    (8, 8, 1, 10000.0, 300), (40, 40, 1, 10000.0, 513), (40, 40, 2, 10000.0, 257), (32, 32, 1, 500000.0, 1024),
    # the widest tensor-core tiles: 11 and 12 FWHT groups per CTA (C = 5632, 6144)
    (44, 44, 4, 10000.0, 90), (48, 48, 4, 10000.0, 130), (48, 48, 1, 10000.0, 70),
    # C = 8192 (16 FWHT groups, one 512-thread CTA per SM); GQA 4:1 at 16 KV heads (generic)
    (64, 64, 4, 10000.0, 70), (64, 64, 2, 10000.0, 33), (64, 16, 2, 500000.0, 70),
    # GQA 4:1 at the paper's G = 4 on the tensor-core kernel (half-group pairs): C = 512 and 1024
    (16, 4, 4, 500000.0, 300), (32, 8, 4, 500000.0, 1025), (32, 8, 4, 10000.0, 1),
    # GQA 8:1 (LLaMA-2/3-70B) and 16:1 as passes of the 4-head kernel, G = 2 and 4
    (64, 8, 2, 500000.0, 300), (64, 8, 4, 500000.0, 129), (32, 4, 2, 10000.0, 77), (64, 4, 4, 10000.0, 65),
    (96, 8, 2, 10000.0, 70), (64, 4, 2, 500000.0, 200), (128, 8, 2, 10000.0, 33),
    # any other ratio: partial head sets (2:1, 3:1 one set; 5:1 .. 7:1 two sets; 10:1 two launches)
    (16, 8, 2, 500000.0, 150), (24, 8, 2, 10000.0, 77), (40, 8, 2, 500000.0, 300), (56, 8, 2, 10000.0, 129),
    (48, 8, 2, 10000.0, 65), (80, 8, 2, 10000.0, 40), (8, 4, 4, 10000.0, 90), (24, 8, 4, 500000.0, 130),
    (20, 4, 4, 10000.0, 33),
    # more than 8 KV heads (5 .. 8 groups per CTA): Phi-3-medium's 40 q / 10 KV, 16 KV heads at G = 2 and 4
    (40, 10, 2, 10000.0, 150), (64, 16, 2, 500000.0, 200), (32, 16, 2, 10000.0, 77), (64, 16, 4, 10000.0, 129),
    (128, 16, 2, 500000.0, 65), (24, 6, 2, 10000.0, 99),  # 6 KV heads: a partial plan store group
    # GQA at the reference's default per-head rotation (G = 1): H_8 x I_2 second factor
    (32, 8, 1, 500000.0, 300), (16, 4, 1, 10000.0, 77), (64, 8, 1, 10000.0, 129), (40, 8, 1, 500000.0, 65),
    (64, 16, 1, 10000.0, 90),
])
def test_decode_vs_oracle(oracle, hq, hkv, g, base, T):
    w = small_workload(hq, hkv, g, base=base)
    B = 2
    layer, perm = build_layer(w, B, T + 8, seed=T)
    k, v = WL.make_kv(w, T, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    if T > 10:
        sinks[0, T // 2] = 1
    layer.append(k, v, sinks)
    q = WL.make_q(w, T, B)
    out = layer.decode(q).cpu().numpy()
    got = cache_host(layer)
    for b in range(B):
        want = oracle_decode(oracle, layer, got, b, T, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(out[b], want) < REL_TOL
        assert cosine(out[b], want) > COS_TOL


@pytest.mark.parametrize("hq,hkv,g,T", [
    (96, 32, 2, 70),    # GQA over 32 KV heads (past the tensor-core GQA width)
    (40, 8, 8, 70),     # 5 q heads per KV head at G = 8
    (64, 64, 1, 90),    # G = 1 at C = 8192
    (16, 16, 8, 130),   # n = 1024
    (32, 32, 16, 65),   # n = 2048
    (64, 64, 64, 40),   # n = 8192 (kMaxHadamardLog2, proj/include/rotatekv/hadamard.hpp:21)
    (24, 8, 8, 50),     # GQA 3:1 at n = 1024
])
def test_generic_shapes_vs_oracle(oracle, hq, hkv, g, T):
    """Shapes the specialised kernels do not tile run on the generic kernels
    (any power-of-two rotation size <= 8192, any head ratio): codes bit-exact,
    decode within the north-star bar of the oracle."""
    w = small_workload(hq, hkv, g)
    B = 2
    layer, perm = build_layer(w, B, T + 4, seed=T + g)
    k, v = WL.make_kv(w, T + g, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    sinks[1, T // 3] = 1
    layer.append(k, v, sinks)
    got = cache_host(layer)
    for b in range(B):
        kc, km, vc, vm = oracle.quantize_kv_rows(k[b].cpu().numpy(), v[b].cpu().numpy(), hkv, 128, g, perm)
        rows = [t for t in range(T) if not sinks[b, t]]
        assert np.array_equal(got["k_codes"][b, rows].view(np.uint32), kc[rows])
        assert np.array_equal(got["k_meta"][b, rows].view(np.uint32), km[rows])
        assert np.array_equal(got["v_codes"][b, rows].view(np.uint32), vc[rows])
        assert np.array_equal(got["v_meta"][b, rows].view(np.uint32), vm[rows])
    q = WL.make_q(w, T + g, B)
    out = layer.decode(q).cpu().numpy()
    for b in range(B):
        want = oracle_decode(oracle, layer, got, b, T, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(out[b], want) < 2e-4, rel_err(out[b], want)  # fp32 dequant: tighter than the bar
        assert cosine(out[b], want) > 0.99999


@pytest.mark.parametrize("hq,hkv,g", [(64, 16, 4), (32, 8, 4), (16, 16, 8)])
def test_generic_tiles_sinks_and_splits(oracle, hq, hkv, g):
    """The tiled generic decode over many tiles and splits: sinks on both sides
    of 32-token mask-word boundaries (a tile's live mask spans two words), a
    sequence with a single sink, and a length that is not a tile multiple."""
    w = small_workload(hq, hkv, g)
    B, T = 3, 1501
    layer, perm = build_layer(w, B, T + 3, seed=5 + g)
    k, v = WL.make_kv(w, 50 + g, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    for t in (31, 32, 63, 64, 95, 1023):
        sinks[1, t] = 1
    sinks[2, 1500] = 1
    layer.append(k, v, sinks)
    got = cache_host(layer)
    q = WL.make_q(w, 60 + g, B)
    out = layer.decode(q).cpu().numpy()
    for b in range(B):
        want = oracle_decode(oracle, layer, got, b, T, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(out[b], want) < 2e-4, (b, rel_err(out[b], want))
        assert cosine(out[b], want) > 0.99999


@pytest.mark.parametrize("hq,hkv,g", [(8, 8, 4), (32, 8, 2), (32, 8, 4)])
def test_decode_sinks_past_the_combine_prefetch(oracle, hq, hkv, g):
    """More sink rows than the combine prefetches (4): rows 0..3 take the
    prefetched path, the rest the per-sink loads; one sequence with none
    past the first and one whose last sink is the final token."""
    w = small_workload(hq, hkv, g)
    B, T = 2, 400
    layer, perm = build_layer(w, B, T + 2, seed=77 + g, max_sinks=8)
    k, v = WL.make_kv(w, 77 + g, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    for t in (0, 5, 31, 32, 200, 333, 399):
        sinks[0, t] = 1
    sinks[1, 0] = 1
    layer.append(k, v, sinks)
    got = cache_host(layer)
    q = WL.make_q(w, 78 + g, B)
    out = layer.decode(q).cpu().numpy()
    for b in range(B):
        want = oracle_decode(oracle, layer, got, b, T, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(out[b], want) < 2e-4, (b, rel_err(out[b], want))
        assert cosine(out[b], want) > 0.99999


@pytest.mark.parametrize("hq,hkv,g", [(8, 8, 4), (16, 4, 2), (16, 4, 4), (16, 16, 8)])
def test_decode_large_batch(oracle, hq, hkv, g):
    """More sequences than resident CTA slots (one split each, several
    waves) and ragged lengths; sampled sequences against the oracle."""
    w = small_workload(hq, hkv, g)
    B, T = 320, 48
    layer, perm = build_layer(w, B, T + 1, seed=400 + g)
    k, v = WL.make_kv(w, 400 + g, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    sinks[::7, 17] = 1
    layer.append(k, v, sinks)
    lens = [T - (b % 13) for b in range(B)]
    q = WL.make_q(w, 401 + g, B)
    out = layer.decode(q, seq_len=lens).cpu().numpy()
    got = cache_host(layer)
    for b in (0, 7, 150, B - 1):
        want = oracle_decode(oracle, layer, got, b, lens[b], q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(out[b], want) < 2e-4, (b, rel_err(out[b], want))
        assert cosine(out[b], want) > 0.99999


def test_generic_decode_matches_reference_decode_step(ref):
    """G = 8 (n = 1024) end to end against the unmodified reference's
    decode_step (e4m3 scales, identity projections)."""
    w = small_workload(16, 16, 8)
    T = 33
    layer, perm = build_layer(w, 1, T + 1, seed=88, fmt=P.SCALE_E4M3_CEIL)
    k, v = WL.make_kv(w, 88, 1, T + 1)
    x = k[:, T:T + 1]
    sinks = torch.zeros(1, T, dtype=torch.uint8)
    sinks[0, 0] = 1
    layer.append(k[:, :T], v[:, :T], sinks)
    out = layer.decode_step(x, x, x.reshape(1, 16, 128)).cpu().numpy().reshape(-1)
    want = ref.ref_decode_step(k[0, :T].float().cpu().numpy(), v[0, :T].float().cpu().numpy(), sinks[0].numpy(),
                               perm, x[0, 0].float().cpu().numpy(), 16, 128, 8, 10000.0)
    assert rel_err(out, want) < REL_TOL
    assert cosine(out, want) > COS_TOL


def test_decode_ragged_lengths(oracle):
    """Sequences of different lengths in one call (split tails, short splits)."""
    w = small_workload(8, 8, 4)
    lens = [1, 17, 64, 251]
    B = len(lens)
    layer, perm = build_layer(w, B, 256, seed=9)
    k, v = WL.make_kv(w, 9, B, 251)
    sinks = torch.zeros(B, 251, dtype=torch.uint8)
    sinks[:, 0] = 1
    sinks[3, 100] = 1
    layer.append(k, v, sinks)
    q = WL.make_q(w, 9, B)
    out = layer.decode(q, seq_len=lens).cpu().numpy()
    got = cache_host(layer)
    for b, T in enumerate(lens):
        want = oracle_decode(oracle, layer, got, b, T, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(out[b], want) < REL_TOL, (b, T)


def test_decode_many_sinks(oracle):
    """More sink tokens than any fixed staging size: 20 sinks in one sequence,
    every one merged into the decode output (no silent cap)."""
    w = small_workload(8, 8, 4)
    B, T = 2, 90
    layer, perm = build_layer(w, B, 96, seed=21, max_sinks=24)
    k, v = WL.make_kv(w, 21, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[0, 0:80:4] = 1  # 20 sinks
    sinks[1, 0] = 1
    layer.append(k, v, sinks)
    q = WL.make_q(w, 21, B)
    out = layer.decode(q).cpu().numpy()
    got = cache_host(layer)
    for b in range(B):
        want = oracle_decode(oracle, layer, got, b, T, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(out[b], want) < REL_TOL, b
        assert cosine(out[b], want) > COS_TOL


def test_decode_step_loop_vs_reference_semantics(oracle):
    """decode_step semantics: append the token, then attend with q at its
    position; several steps, each checked against the oracle."""
    w = small_workload(8, 8, 4)
    B, T0 = 2, 50
    layer, perm = build_layer(w, B, 64, seed=12)
    k, v = WL.make_kv(w, 12, B, T0 + 4)
    sinks = torch.zeros(B, T0, dtype=torch.uint8)
    sinks[:, 0] = 1
    layer.append(k[:, :T0], v[:, :T0], sinks)
    for step in range(4):
        t = T0 + step
        q = WL.make_q(w, 12, B, step=step)
        out = layer.decode_step(k[:, t:t + 1], v[:, t:t + 1], q).cpu().numpy()
        got = cache_host(layer)
        for b in range(B):
            want = oracle_decode(oracle, layer, got, b, t + 1, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                                 v[b].cpu().numpy())
            assert rel_err(out[b], want) < REL_TOL


def test_decode_matches_reference_decode_step(ref):
    """End to end against the reference's own decode_step
    (proj/src/pipeline.cpp:193-263) in e4m3 mode, identity projections."""
    w = small_workload(8, 8, 4)
    T = 40
    layer, perm = build_layer(w, 1, T + 1, seed=21, fmt=P.SCALE_E4M3_CEIL)
    k, v = WL.make_kv(w, 21, 1, T + 1)
    x = k[:, T:T + 1]  # decode token: key = value = query (identity W)
    sinks = torch.zeros(1, T, dtype=torch.uint8)
    sinks[0, 0] = 1
    sinks[0, 11] = 1
    layer.append(k[:, :T], v[:, :T], sinks)
    out = layer.decode_step(x, x, x.reshape(1, 8, 128)).cpu().numpy().reshape(-1)
    want = ref.ref_decode_step(k[0, :T].float().cpu().numpy(), v[0, :T].float().cpu().numpy(), sinks[0].numpy(),
                               perm, x[0, 0].float().cpu().numpy(), 8, 128, 4, 10000.0)
    assert rel_err(out, want) < REL_TOL
    assert cosine(out, want) > COS_TOL


@pytest.mark.parametrize("hq,hkv,g", [(40, 40, 4), (32, 8, 2), (32, 8, 4), (16, 16, 8), (64, 32, 1), (64, 8, 2),
                                      (40, 8, 2), (32, 8, 1)])
def test_decode_deterministic(hq, hkv, g):
    """Bit-identical outputs run to run on every decode kernel family (fixed
    split partition, fixed merge order)."""
    w = small_workload(hq, hkv, g)
    layer, perm = build_layer(w, 2, 600, seed=4)
    k, v = WL.make_kv(w, 4, 2, 600)
    layer.append(k, v)
    q = WL.make_q(w, 4, 2)
    a = layer.decode(q).clone()
    for _ in range(20):
        assert torch.equal(a, layer.decode(q))


@pytest.mark.parametrize("cfg_id", [2, 3, 4])
def test_full_size_decode_sampled_vs_oracle(oracle, cfg_id):
    """BASELINE config sizes: the whole batch runs on the GPU; two sampled
    sequences are checked against the oracle (cfg3: one 8-sequence shard of
    the 64; cfg4: the 32768-token context of one GPU's 1-sequence shard,
    plus a second sequence)."""
    w = WL.CONFIGS[cfg_id]
    B = {2: w.batch, 3: 8, 4: 2}[cfg_id]
    T = w.tokens
    layer, perm = build_layer(w, B, T + 1, seed=cfg_id)
    k, v = WL.make_kv(w, cfg_id, B, T)
    flags = torch.zeros(B, T, dtype=torch.uint8)
    for t in WL.sink_positions(w, cfg_id, T):
        flags[:, t] = 1
    layer.append(k, v, flags)
    q = WL.make_q(w, cfg_id, B)
    out = layer.decode(q).cpu().numpy()
    got = cache_host(layer)
    for b in (0, B - 1):
        want = oracle_decode(oracle, layer, got, b, T, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(out[b], want) < REL_TOL
        assert cosine(out[b], want) > COS_TOL


def test_full_size_quantize_sampled_rows_bit_exact(oracle):
    """cfg2-sized append; sampled rows checked bit-exact."""
    w = WL.CONFIGS[2]
    B, T = 16, 1024
    layer, perm = build_layer(w, B, T, seed=22)
    k, v = WL.make_kv(w, 22, B, T)
    layer.append(k, v)
    got = cache_host(layer)
    rng = np.random.default_rng(0)
    for b in rng.choice(B, 3, replace=False):
        rows = np.sort(rng.choice(T, 16, replace=False))
        kc, km, vc, vm = oracle.quantize_kv_rows(k[b, rows].cpu().numpy(), v[b, rows].cpu().numpy(), 40, 128, 4,
                                                 perm)
        assert np.array_equal(got["k_codes"][b, rows].view(np.uint32), kc)
        assert np.array_equal(got["k_meta"][b, rows].view(np.uint32), km)
        assert np.array_equal(got["v_codes"][b, rows].view(np.uint32), vc)
        assert np.array_equal(got["v_meta"][b, rows].view(np.uint32), vm)


def test_rotate_keys_matches_oracle(oracle):
    w = small_workload(8, 8, 4)
    cfg = P.LayerConfig(batch=1, num_q_heads=8, num_kv_heads=8, heads_per_group=4)
    k, _ = WL.make_kv(w, 30, 1, 16)
    got = P.rotate_keys(cfg, k[0]).cpu().numpy()
    want = oracle.rotate_rows(k[0].float().cpu().numpy(), 128, 4, 8)
    assert np.array_equal(got, want)


def test_errors_mirror_reference_exceptions():
    w = small_workload(8, 8, 4)
    layer, perm = build_layer(w, 1, 8, seed=1, max_sinks=1)
    k, v = WL.make_kv(w, 1, 1, 9)
    with pytest.raises(IndexError):  # std::out_of_range: past capacity
        layer.append(k, v)
    with pytest.raises(ValueError):  # std::invalid_argument: row length
        layer.append(k[:, :, :512], v[:, :, :512])
    two = torch.ones(1, 2, dtype=torch.uint8)
    with pytest.raises(IndexError):  # sidecar full
        layer.append(k[:, :2], v[:, :2], two)
    with pytest.raises(ValueError):  # position must equal current cache length
        layer.decode(WL.make_q(w, 1, 1))


def test_cpp_api_program(tmp_path):
    """The C++ API (rotatekv.hpp) end to end: parity + exception classes."""
    import subprocess

    from tests._cpp import build_cpp_test

    exe = build_cpp_test(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.fixture
def debug_option():
    """Set an experiment switch for one test and restore the default after."""
    import paper_2501_16383_b200 as P

    defaults = {"gqa_tmem": 1, "decode_kernel_simt": 0, "prefill_pair": 0, "decode_splits": 0, "gqa_warps_per_group": 1,
                "gqa_head_sets": 2, "quant_stages": 1, "quant_vsplit": 1, "quant_vcfg": 0}
    touched = []

    def set_(name, value):
        touched.append(name)
        P.set_debug_option(name, value)

    yield set_
    for name in touched:
        P.set_debug_option(name, defaults[name])


@pytest.mark.parametrize("opt,hq,hkv,g", [("gqa_tmem=0", 32, 8, 2), ("decode_kernel_simt=1", 8, 8, 4),
                                          ("decode_kernel_simt=1", 32, 8, 2), ("gqa_warps_per_group=2", 32, 8, 2),
                                          ("gqa_warps_per_group=2", 32, 8, 4), ("gqa_warps_per_group=4", 32, 8, 2),
                                          ("gqa_head_sets=1", 64, 8, 2), ("gqa_tmem=0", 64, 8, 2),
                                          ("gqa_warps_per_group=2", 64, 8, 2)])
def test_alternative_decode_kernels(oracle, debug_option, opt, hq, hkv, g):
    """The switch-selectable kernels (register-resident GQA, the CUDA-core
    kernel on tensor-core shapes) stay parity-green.  The layer (plan and RoPE
    table layout) is built under the same selection."""
    k_, v_ = opt.split("=")
    debug_option(k_, int(v_))
    w = small_workload(hq, hkv, g)
    B, T = 2, 150
    layer, perm = build_layer(w, B, T + 8, seed=77)
    k, v = WL.make_kv(w, 77, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    layer.append(k, v, sinks)
    q = WL.make_q(w, 77, B)
    out = layer.decode(q).cpu().numpy()
    got = cache_host(layer)
    for b in range(B):
        want = oracle_decode(oracle, layer, got, b, T, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(out[b], want) < REL_TOL
        assert cosine(out[b], want) > COS_TOL


@pytest.mark.parametrize("opt,hq,hkv,g", [("quant_stages=2", 40, 40, 4), ("quant_stages=2", 64, 64, 2),
                                          ("quant_vsplit=0", 32, 32, 4), ("quant_vsplit=0", 8, 8, 4),
                                          ("quant_vcfg=3", 40, 40, 4), ("quant_vcfg=4", 32, 32, 2),
                                          ("quant_vcfg=1", 40, 40, 4)])
def test_alternative_quantize_kernels(oracle, debug_option, opt, hq, hkv, g):
    """The switch-selectable quantize variants stay bit-exact (enough token
    pairs that the V kernel split and several items per CTA engage)."""
    k_, v_ = opt.split("=")
    debug_option(k_, int(v_))
    w = small_workload(hq, hkv, g)
    B, T = 8, 333
    layer, perm = build_layer(w, B, T, seed=41)
    k, v = WL.make_kv(w, 41, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    sinks[3, 100] = 1
    layer.append(k, v, sinks)
    torch.cuda.synchronize()
    got = cache_host(layer)
    for b in (0, 3, B - 1):
        kc, km, vc, vm = oracle.quantize_kv_rows(k[b].cpu().numpy(), v[b].cpu().numpy(), hkv, 128, g, perm)
        rows = [t for t in range(T) if not sinks[b, t]]
        assert np.array_equal(got["k_codes"][b, rows].view(np.uint32), kc[rows])
        assert np.array_equal(got["k_meta"][b, rows].view(np.uint32), km[rows])
        assert np.array_equal(got["v_codes"][b, rows].view(np.uint32), vc[rows])
        assert np.array_equal(got["v_meta"][b, rows].view(np.uint32), vm[rows])


@pytest.mark.parametrize("hq,hkv,g", [(64, 8, 2), (32, 4, 2), (128, 8, 2), (40, 8, 2), (56, 8, 2)])
def test_gqa_head_sets_bit_identical_to_passes(debug_option, hq, hkv, g):
    """Two 4-head sets per key tile (the 8:1 default) run each head's
    arithmetic exactly as the 4-head passes do: the outputs are bit-identical."""
    w = small_workload(hq, hkv, g)
    B, T = 3, 300
    layer, perm = build_layer(w, B, T + 4, seed=61)
    k, v = WL.make_kv(w, 61, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    layer.append(k, v, sinks)
    q = WL.make_q(w, 61, B)
    sets = layer.decode(q).cpu().numpy()
    debug_option("gqa_head_sets", 1)
    passes = layer.decode(q).cpu().numpy()
    assert np.array_equal(sets.view(np.uint32), passes.view(np.uint32))
