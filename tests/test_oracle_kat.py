"""Pin the CPU restatement (oracle/rkv_oracle.c) on the reference's own
known-answer tests.  Each test cites the reference test it restates
(/root/reference/proj/tests/...).  CPU only."""
import math

import numpy as np
import pytest


def test_two_bit_example_quantizes_exactly(oracle):
    # proj/tests/test_quant.cpp:11-23
    for fmt in (oracle.SCALE_E4M3_CEIL, oracle.SCALE_FP16_CEIL):
        s, z, codes, _ = oracle.quantize_group([-1, 0, 1, 2], 2, fmt)
        assert s == 1.0 and z == 1 and list(codes) == [0, 1, 2, 3]


def test_non_negative_ramp_has_zero_point_0(oracle):
    # proj/tests/test_quant.cpp:25-34
    for fmt in (oracle.SCALE_E4M3_CEIL, oracle.SCALE_FP16_CEIL):
        s, z, codes, _ = oracle.quantize_group([0, 1, 2, 3], 2, fmt)
        assert s == 1.0 and z == 0 and list(codes) == [0, 1, 2, 3]


def test_constant_group(oracle):
    # proj/tests/test_quant.cpp:36-51
    for fmt in (oracle.SCALE_E4M3_CEIL, oracle.SCALE_FP16_CEIL):
        s, z, codes, _ = oracle.quantize_group([5, 5, 5, 5], 2, fmt)
        assert len(set(codes.tolist())) == 1 and s >= 1e-8
        s, z, codes, _ = oracle.quantize_group([0, 0, 0, 0], 2, fmt)
        back = np.float32(s) * (codes.astype(np.float32) - np.float32(z))
        assert np.all(np.abs(back) < 1e-6)


def test_pack_unpack_round_trip(oracle):
    # proj/tests/test_quant.cpp:53-66
    rng = np.random.default_rng(31)
    for bits in (2, 3, 4):
        length = 1
        while length <= 256:
            codes = rng.integers(0, 1 << bits, length).astype(np.uint8)
            packed = oracle.pack_codes(codes, bits)
            assert packed.size == (length * bits + 7) // 8
            assert np.array_equal(oracle.unpack_codes(packed, length, bits), codes)
            length += 1 if length < 16 else 17


def test_lsb_first_packing_equals_u32_words(oracle):
    # proj/src/quant.cpp:25-35 byte order == code i at bits 2*(i%16) of LE word i/16
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 4, 128).astype(np.uint8)
    words = oracle.pack_codes(codes, 2).view("<u4")
    for i in range(128):
        assert (int(words[i // 16]) >> (2 * (i % 16))) & 3 == codes[i]


@pytest.mark.parametrize("fmt", [0, 1])
def test_reconstruction_error_bound(oracle, fmt):
    # proj/tests/test_quant.cpp:91-105 (bits 3, group 64)
    rng = np.random.default_rng(33)
    for _ in range(200):
        x = (rng.standard_normal(64) * 7).astype(np.float32)
        s, z, codes, _ = oracle.quantize_group(x, 3, fmt)
        back = np.float32(s) * (codes.astype(np.float32) - np.float32(z))
        assert np.all(np.abs(x - back) <= s * (0.5 + 1.0 / 16.0) + 1e-6)


@pytest.mark.parametrize("fmt", [0, 1])
def test_requantize_reproduces_codes(oracle, fmt):
    # proj/tests/test_quant.cpp:107-124
    rng = np.random.default_rng(34)
    x = (rng.standard_normal(32) * 3).astype(np.float32)
    s, z, codes, _ = oracle.quantize_group(x, 2, fmt)
    back = np.float32(s) * (codes.astype(np.float32) - np.float32(z))
    again = np.clip(np.round(back.astype(np.float64) / s) + z, 0, 3).astype(np.uint8)
    assert np.array_equal(again, codes)


def test_mse_non_increasing_in_bits(oracle):
    # proj/tests/test_quant.cpp:126-142
    rng = np.random.default_rng(35)
    x = (rng.standard_normal(128) * 2).astype(np.float32)
    prev = 1e30
    for bits in (2, 3, 4, 5, 6):
        s, z, codes, _ = oracle.quantize_group(x, bits, oracle.SCALE_E4M3_CEIL)
        back = np.float32(s) * (codes.astype(np.float32) - np.float32(z))
        err = float(np.sum((x - back).astype(np.float64) ** 2))
        assert err <= prev * 1.0001
        prev = err


def test_e4m3_known_values(oracle):
    # proj/tests/test_fp8.cpp:10-19
    d = oracle.e4m3_decode
    assert d(0x00) == 0.0 and d(0x38) == 1.0 and d(0x7E) == 448.0
    assert d(0x08) == pytest.approx(2.0 ** -6) and d(0x01) == pytest.approx(2.0 ** -9)
    assert math.isnan(d(0x7F)) and math.isnan(d(0xFF)) and d(0xB8) == -1.0


def test_e4m3_monotone_and_round_trip(oracle):
    # proj/tests/test_fp8.cpp:21-33
    for c in range(0x7E):
        assert oracle.e4m3_decode(c) < oracle.e4m3_decode(c + 1)
    for c in range(0xFF):
        if (c & 0x7F) == 0x7F or c == 0x80:
            continue
        assert oracle.e4m3_encode(oracle.e4m3_decode(c)) == c


def test_e4m3_ties_to_even(oracle):
    # proj/tests/test_fp8.cpp:35-43
    e = oracle.e4m3_encode
    assert e(1.0625) == 0x38 and e(1.1875) == 0x3A and e(1.06) == 0x38
    assert e(1.07) == 0x39 and e(1000.0) == 0x7E


def test_e4m3_encode_ceil(oracle):
    # proj/tests/test_fp8.cpp:45-56
    rng = np.random.default_rng(7)
    for v in np.exp(rng.standard_normal(2000) * 3.0):
        x = np.float32(min(v, 448.0))
        code = oracle.e4m3_encode_ceil(x)
        assert oracle.e4m3_decode(code) >= x
        if code > 0:
            assert oracle.e4m3_decode(code - 1) < x
    assert oracle.e4m3_decode(oracle.e4m3_encode_ceil(1.0)) == 1.0


def test_fp16_ceil_is_smallest_fp16_at_or_above(oracle):
    # fp16 analogue of proj/tests/test_fp8.cpp:45-56
    rng = np.random.default_rng(8)
    xs = np.exp(rng.standard_normal(4000) * 6.0).astype(np.float32)
    xs = np.concatenate([xs, np.float32([1e-8, 6e-8, 1.0, 65504.0, 1e5, 2.0 ** -14])])
    for x in xs:
        h = oracle.fp16_ceil(x)
        v = np.uint16(h).view(np.float16).astype(np.float32)
        if x <= 65504.0:
            assert v >= x
            if h > 0:
                assert np.uint16(h - 1).view(np.float16).astype(np.float32) < x
        else:
            assert h == 0x7BFF  # saturates like proj/src/fp8.cpp:71
    # exact fp16 values stay exact
    for v in np.float16([1.0, 0.5, 3.0, 1e-4, 60000.0]):
        assert oracle.fp16_ceil(np.float32(v)) == np.float16(v).view(np.uint16)


def test_float_to_half_matches_numpy(oracle):
    rng = np.random.default_rng(9)
    xs = np.concatenate([rng.standard_normal(3000) * 10.0 ** rng.integers(-9, 6, 3000),
                         [0.0, -0.0, 65519.0, 65520.0, 2.0 ** -25, 3 * 2.0 ** -26, 1e-30]]).astype(np.float32)
    for x in xs:
        assert oracle.float_to_half(x) == np.float16(x).view(np.uint16), x
        h = np.float16(x)
        assert oracle.half_to_float(h.view(np.uint16)) == np.float32(h)


def test_fwht_oracle_n4(oracle):
    # proj/tests/test_hadamard.cpp:37-41
    assert np.allclose(oracle.fwht([1, 0, 0, 0]), 0.5)


def test_fwht_involutory(oracle):
    # proj/tests/test_hadamard.cpp:43-50
    rng = np.random.default_rng(3)
    v = (rng.standard_normal(128) * 10).astype(np.float32)
    assert np.allclose(oracle.fwht(oracle.fwht(v)), v, rtol=1e-5, atol=1e-5)


def test_fwht_matches_explicit_matrix(oracle):
    # proj/tests/acceptance.cpp:37-62 (criterion 1, n = 2..4096, < 1e-5)
    rng = np.random.default_rng(4)
    for k in range(1, 13):
        n = 1 << k
        h = np.array([[(-1) ** bin(i & j).count("1") for j in range(n)] for i in range(n)]) / math.sqrt(n) if n <= 512 else None
        v = rng.standard_normal(n).astype(np.float32)
        got = oracle.fwht(v)
        if h is not None:
            assert np.max(np.abs(got - h @ v.astype(np.float64))) < 1e-5
        assert np.allclose(np.linalg.norm(got), np.linalg.norm(v), rtol=1e-5)


def test_fwht_rejects_non_power_of_two(oracle):
    # proj/tests/test_hadamard.cpp:52-55
    with pytest.raises(ValueError):
        oracle.fwht([1, 2, 3])


def test_rotation_plan_validation(oracle):
    # proj/tests/test_hadamard.cpp:57-61
    for d, g, h in ((96, 1, 8), (128, 3, 8), (8192, 2, 2)):
        with pytest.raises(ValueError):
            oracle.rotate_rows(np.zeros(d * h, np.float32), d, g, h)


def test_grouped_rotation_norm_and_per_head(oracle):
    # proj/tests/test_hadamard.cpp:63-100
    rng = np.random.default_rng(11)
    x = rng.standard_normal((6, 64)).astype(np.float32)
    y = oracle.rotate_rows(x, 16, 2, 4)
    assert np.allclose(np.linalg.norm(y, axis=1), np.linalg.norm(x, axis=1), rtol=1e-5)
    assert np.allclose(oracle.rotate_rows(y, 16, 2, 4), x, rtol=1e-5, atol=1e-6)
    z = oracle.rotate_rows(x, 16, 1, 4)
    for h in range(4):
        for r in range(6):
            assert np.allclose(z[r, h * 16:(h + 1) * 16], oracle.fwht(x[r, h * 16:(h + 1) * 16]), atol=1e-6)


def test_calibrate_ascending_argsort(oracle):
    # proj/tests/test_reorder.cpp:22-30
    perm, inv = oracle.calibrate_reorder(np.float32([[3.0, -5.0, 1.0]]))
    assert list(perm) == [1, 2, 0] and inv[1] == 0 and inv[2] == 1 and inv[0] == 2


def test_calibrate_stable_ties(oracle):
    # proj/tests/test_reorder.cpp:32-36
    perm, _ = oracle.calibrate_reorder(np.float32([[1, 1, 1, 1], [-1, -1, -1, -1]]))
    assert list(perm) == [0, 1, 2, 3]


def test_calibrate_token_order_independent(oracle):
    # proj/tests/test_reorder.cpp:38-42
    a = np.float32([[1, 5, -2, 0], [2, -1, 3, 1], [0, 0, 1, -4]])
    b = np.float32([[0, 0, 1, -4], [1, 5, -2, 0], [2, -1, 3, 1]])
    assert np.array_equal(oracle.calibrate_reorder(a)[0], oracle.calibrate_reorder(b)[0])


def test_calibrate_mean_abs_statistic(oracle):
    # mean |K| variant used for the BASELINE configs
    x = np.float32([[3, -5, 1], [-3, 5, 1]])
    perm, _ = oracle.calibrate_reorder(x, oracle.STAT_MEAN_ABS)
    assert list(perm) == [2, 0, 1]


def test_reorder_round_trip_bit_exact(oracle):
    # proj/tests/test_reorder.cpp:53-66
    rng = np.random.default_rng(42)
    x = rng.standard_normal((7, 12)).astype(np.float32)
    perm, _ = oracle.calibrate_reorder(rng.standard_normal((1, 12)).astype(np.float32))
    y = oracle.apply_reorder(x, perm)
    assert np.array_equal(oracle.apply_reorder(y, perm, inverse=True), x)
    assert np.array_equal(oracle.apply_reorder(x, np.arange(12)), x)


def test_rope_position_zero_identity(oracle):
    # proj/tests/test_rope.cpp:20-28
    rng = np.random.default_rng(21)
    x = rng.standard_normal((3, 16)).astype(np.float32)
    assert np.array_equal(oracle.apply_rope_rows(x, 2, 8, 10000.0, [0, 0, 0]), x)


def test_rope_d2_unit_rotation(oracle):
    # proj/tests/test_rope.cpp:30-37
    y = oracle.apply_rope_rows(np.float32([[1.0, 0.0]]), 1, 2, 10000.0, [1])
    assert y[0, 0] == pytest.approx(math.cos(1.0)) and y[0, 1] == pytest.approx(math.sin(1.0))


def test_rope_inverse_and_relative_position(oracle):
    # proj/tests/test_rope.cpp:55-61 and :80-99
    rng = np.random.default_rng(23)
    x = rng.standard_normal((5, 64)).astype(np.float32)
    pos = [0, 3, 7, 11, 100]
    y = oracle.apply_rope_rows(oracle.apply_rope_rows(x, 2, 32, 10000.0, pos), 2, 32, 10000.0, pos, inverse=True)
    assert np.allclose(y, x, rtol=1e-6, atol=1e-6)
    q = rng.standard_normal((1, 64)).astype(np.float32)
    k = rng.standard_normal((1, 64)).astype(np.float32)

    def dot(mq, mk):
        return float(np.dot(oracle.apply_rope_rows(q, 1, 64, 10000.0, [mq])[0].astype(np.float64),
                            oracle.apply_rope_rows(k, 1, 64, 10000.0, [mk])[0]))

    assert dot(7, 3) == pytest.approx(dot(27, 23), rel=1e-5)
    assert dot(12, 0) == pytest.approx(dot(112, 100), rel=1e-5)


def _block_with_spikes(s, hidden, spikes, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((1, s, hidden)).astype(np.float32)
    for t, c, m in spikes:
        x[0, t, c] = m
    return x


def test_sink_detection(oracle):
    # proj/tests/test_sink.cpp:16-32, :34-41, :43-51, :53-58, :67-79
    x = _block_with_spikes(128, 4096, [(0, 1415, 100.0), (110, 2533, 100.0)])
    assert np.flatnonzero(oracle.detect_sinks(x)).tolist() == [0, 110]
    assert np.flatnonzero(oracle.detect_sinks(_block_with_spikes(64, 256, []))).tolist() == [0]
    assert np.flatnonzero(oracle.detect_sinks(_block_with_spikes(64, 256, [(20, 100, 5.0)]))).tolist() == [0]
    assert np.flatnonzero(oracle.detect_sinks(np.full((1, 1, 16), 0.1, np.float32))).tolist() == [0]
    x = _block_with_spikes(96, 512, [(7, 31, 120.0)])
    assert np.array_equal(oracle.detect_sinks(x), oracle.detect_sinks(x * np.float32(3.7)))
    with pytest.raises(ValueError):
        oracle.detect_sinks(np.zeros((1, 4, 8), np.float32), rel=1.0)


def _dense_reference(kr, vr, q, hq, hkv, d, base):
    """float64 numpy attention for all-sink (unquantized) caches."""
    T = kr.shape[0]
    kpos = np.arange(T)

    def rope(x, pos):
        half = d // 2
        th = base ** (-2.0 * np.arange(half) / d)
        ang = pos[:, None] * th[None]
        c, s = np.cos(ang), np.sin(ang)
        x = x.reshape(x.shape[0], -1, d).astype(np.float64)
        a, b = x[..., :half], x[..., half:]
        return np.concatenate([a * c[:, None] - b * s[:, None], a * s[:, None] + b * c[:, None]], -1)

    k = rope(kr, kpos)
    qq = rope(q.reshape(1, -1), np.array([T - 1]))[0]
    v = vr.reshape(T, hkv, d).astype(np.float64)
    out = np.empty((hq, d))
    for h in range(hq):
        kv = h // (hq // hkv)
        lg = k[:, kv] @ qq[h] / math.sqrt(d)
        p = np.exp(lg - lg.max())
        p /= p.sum()
        out[h] = p @ v[:, kv]
    return out


def test_decode_all_sinks_is_exact_attention(oracle):
    # Decode over a cache whose every token is kept in fp16 (proj/tests/
    # test_kv_cache.cpp:22-45 exact sink bypass) equals plain RoPE attention.
    rng = np.random.default_rng(61)
    hq, hkv, d, g, T = 4, 2, 128, 2, 9
    c = hkv * d
    k = rng.standard_normal((T, c)).astype(np.float16)
    v = rng.standard_normal((T, c)).astype(np.float16)
    q = rng.standard_normal(hq * d).astype(np.float16)
    perm = rng.permutation(c)
    z = np.zeros((T, c // 16), np.uint32)
    m = np.zeros((T, c // 128), np.uint32)
    out = oracle.decode_attention(z, m, z, m, np.ones(T, np.uint8), k, v, q, hq, hkv, d, g, perm, 10000.0)
    ref = _dense_reference(k.astype(np.float32), v.astype(np.float32), q.astype(np.float32), hq, hkv, d, 10000.0)
    assert np.max(np.abs(out - ref)) / np.max(np.abs(ref)) < 1e-5


def test_decode_single_token_returns_value(oracle):
    # softmax of a singleton is one (proj/tests/test_pipeline.cpp:192-196)
    rng = np.random.default_rng(62)
    d, h = 128, 2
    c = h * d
    k = rng.standard_normal((1, c)).astype(np.float16)
    v = rng.standard_normal((1, c)).astype(np.float16)
    q = rng.standard_normal(c).astype(np.float16)
    z = np.zeros((1, c // 16), np.uint32)
    m = np.zeros((1, c // 128), np.uint32)
    out = oracle.decode_attention(z, m, z, m, np.ones(1, np.uint8), k, v, q, h, h, d, 1, np.arange(c), 10000.0)
    assert np.allclose(out.reshape(-1), v.astype(np.float32).reshape(-1), atol=1e-5)
