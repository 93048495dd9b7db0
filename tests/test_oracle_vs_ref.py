"""Pin the CPU restatement against the UNMODIFIED reference library
(oracle/_ref, compiled from /root/reference/proj/src by oracle/Makefile).
Skipped where _ref was never built.  CPU only."""
import numpy as np
import pytest


def _adversarial_groups(rng, n_groups):
    """Random groups plus groups whose values sit exactly on rounding
    boundaries (x = (m - 0.5) * s) of the scale the group will get."""
    out = []
    for i in range(n_groups):
        scale = rng.choice([1e-6, 1e-3, 0.1, 1.0, 7.0, 100.0, 3000.0])
        x = (rng.standard_normal(128) * scale).astype(np.float32)
        if i % 3 == 0:  # plant boundary values
            lo, hi = float(x.min()), float(x.max())
            s = (hi - lo) / 3.0
            ks = rng.integers(-3, 4, 16)
            x[rng.integers(0, 128, 16)] = ((ks - 0.5) * s).astype(np.float32)
            x = np.clip(x, lo, hi).astype(np.float32)
        if i % 7 == 0:
            x[:] = np.float32(scale)  # constant group
        out.append(x)
    return out


def test_quantize_group_e4m3_bit_exact(ref):
    rng = np.random.default_rng(1)
    for x in _adversarial_groups(rng, 3000):
        s, z, codes, sc = ref.quantize_group(x, 2, ref.SCALE_E4M3_CEIL)
        rs, rz, rcodes, rpacked = ref.ref_quantize_group(x, 2, 128)
        assert (sc, z) == (rs, rz)
        assert np.array_equal(codes, rcodes)
        assert np.array_equal(ref.pack_codes(codes, 2), rpacked)


@pytest.mark.parametrize("bits", [1, 3, 4, 8])
def test_quantize_group_other_widths(ref, bits):
    rng = np.random.default_rng(bits)
    for n in (1, 5, 64, 100):
        x = (rng.standard_normal(n) * 5).astype(np.float32)
        s, z, codes, sc = ref.quantize_group(x, bits, ref.SCALE_E4M3_CEIL)
        rs, rz, rcodes, _ = ref.ref_quantize_group(x, bits, 128)
        assert (sc, z) == (rs, rz) and np.array_equal(codes, rcodes)


def test_e4m3_codec_exhaustive(ref):
    for c in range(256):
        a, b = ref.e4m3_decode(c), ref.e4m3_decode(c, impl="ref")
        assert (np.isnan(a) and np.isnan(b)) or a == b
    rng = np.random.default_rng(2)
    for x in np.concatenate([np.exp(rng.standard_normal(5000) * 4), [0.0, 448.0, 500.0, 2.0 ** -10]]):
        x = np.float32(x)
        assert ref.e4m3_encode(x) == ref.e4m3_encode(x, impl="ref")
        assert ref.e4m3_encode_ceil(x) == ref.e4m3_encode_ceil(x, impl="ref")


@pytest.mark.parametrize("n", [2, 16, 128, 256, 512, 1024, 8192])
def test_fwht_bit_exact(ref, n):
    rng = np.random.default_rng(n)
    v = (rng.standard_normal(n) * 30).astype(np.float32)
    assert np.array_equal(ref.fwht(v), ref.fwht(v, impl="ref"))


@pytest.mark.parametrize("h,d,g", [(32, 128, 4), (40, 128, 4), (8, 128, 2), (4, 128, 1)])
def test_rotate_and_reorder_bit_exact(ref, h, d, g):
    rng = np.random.default_rng(h * g)
    x = rng.standard_normal((5, h * d)).astype(np.float32)
    assert np.array_equal(ref.rotate_rows(x, d, g, h), ref.rotate_rows(x, d, g, h, impl="ref"))
    perm = rng.permutation(h * d).astype(np.int32)
    for inv in (False, True):
        assert np.array_equal(ref.apply_reorder(x, perm, inv), ref.apply_reorder(x, perm, inv, impl="ref"))


def test_calibrate_reorder_matches(ref):
    rng = np.random.default_rng(3)
    for c in (12, 1024, 4096):
        x = rng.standard_normal((64, c)).astype(np.float32)
        x[:, rng.integers(0, c, 8)] *= 20
        a = ref.calibrate_reorder(x)
        b = ref.calibrate_reorder(x, impl="ref")
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("base", [10000.0, 500000.0])
def test_rope_bit_exact(ref, base):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((6, 256)).astype(np.float32)
    pos = [0, 1, 17, 4095, 8191, 32767]
    for inv in (False, True):
        assert np.array_equal(ref.apply_rope_rows(x, 2, 128, base, pos, inv),
                              ref.apply_rope_rows(x, 2, 128, base, pos, inv, impl="ref"))


def test_sink_detection_matches(ref):
    rng = np.random.default_rng(5)
    for s, h in ((64, 256), (300, 512)):
        x = rng.standard_normal((2, s, h)).astype(np.float32)
        for t in rng.integers(0, s, 3):
            x[rng.integers(0, 2), t, rng.integers(0, h)] = 100.0
        assert np.array_equal(ref.detect_sinks(x), ref.detect_sinks(x, impl="ref"))


@pytest.mark.parametrize("h,g", [(8, 4), (8, 2), (4, 1)])
def test_quantize_kv_rows_e4m3_bit_exact(ref, h, g):
    d = 128
    c = h * d
    rng = np.random.default_rng(6 + g)
    k = rng.standard_normal((24, c)).astype(np.float16)
    k[:, rng.integers(0, c, 6)] *= np.float16(20)
    v = rng.standard_normal((24, c)).astype(np.float16)
    perm = rng.permutation(c).astype(np.int32)
    kc, km, vc, vm = ref.quantize_kv_rows(k, v, h, d, g, perm, ref.SCALE_E4M3_CEIL)
    rkc, rks, rkz, rvc, rvs, rvz = ref.ref_quantize_kv_rows(k.astype(np.float32), v.astype(np.float32), h, d, g, perm)
    assert np.array_equal(kc, rkc) and np.array_equal(vc, rvc)
    dec = np.vectorize(lambda s: ref.e4m3_decode(int(s)))
    assert np.array_equal((km & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float32), dec(rks).astype(np.float32))
    assert np.array_equal((km >> 16).astype(np.uint16).view(np.float16).astype(np.float32), rkz.astype(np.float32))
    assert np.array_equal((vm & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float32), dec(rvs).astype(np.float32))


@pytest.mark.parametrize("h,g,T,base", [(8, 4, 40, 10000.0), (4, 2, 70, 500000.0), (4, 1, 5, 10000.0)])
def test_decode_matches_reference_decode_step(ref, h, g, T, base):
    """The oracle's decode over an e4m3 cache vs the reference's own
    decode_step (proj/src/pipeline.cpp:193-263) on identical inputs."""
    d = 128
    c = h * d
    rng = np.random.default_rng(T)
    k = rng.standard_normal((T, c)).astype(np.float16)
    k[:, rng.integers(0, c, 4 * h)] *= np.float16(15)
    v = rng.standard_normal((T, c)).astype(np.float16)
    x = rng.standard_normal(c).astype(np.float16)
    sink = np.zeros(T, np.uint8)
    sink[0] = 1
    sink[T // 3] = 1
    perm = rng.permutation(c).astype(np.int32)
    want = ref.ref_decode_step(k.astype(np.float32), v.astype(np.float32), sink, perm, x.astype(np.float32), h, d, g, base)
    K = np.concatenate([k, x[None]])
    V = np.concatenate([v, x[None]])
    S = np.concatenate([sink, [0]]).astype(np.uint8)
    kc, km, vc, vm = ref.quantize_kv_rows(K, V, h, d, g, perm, ref.SCALE_E4M3_CEIL)
    got = ref.decode_attention(kc, km, vc, vm, S, K, V, x, h, h, d, g, perm, base).reshape(-1)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-4
