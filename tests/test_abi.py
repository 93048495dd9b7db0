"""The C-ABI library (CPU-side checks, no GPU): it loads, exports every
symbol include/rotatekv/rotatekv.h declares, and its host-only entry points
validate like the reference and compute like the oracle."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2501_16383_b200 as P
from paper_2501_16383_b200 import rotatekv as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2501_16383_b200 import build

    build.build()
    return R.lib()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "rotatekv", "rotatekv.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w ]+?\*?\s*\b(rkv_\w+)\s*\(", text, re.M)))


def test_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", R.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s+(rkv_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert hasattr(lib, s)


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", R.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version(lib):
    assert b"sm_100a" in lib.rkv_version()


def cfg(**kw):
    base = dict(batch=2, num_q_heads=8, num_kv_heads=8, heads_per_group=4, max_tokens=64)
    base.update(kw)
    return P.LayerConfig(**base)


@pytest.mark.parametrize("kw,msg", [
    (dict(heads_per_group=3), "heads_per_group must divide num_heads"),   # proj/tests/test_hadamard.cpp:59
    (dict(num_kv_heads=6, num_q_heads=6, heads_per_group=3), "power of two"),
    (dict(bits=0), "quant bits must be in [1,8]"),                          # proj/tests/test_quant.cpp:188-191
    (dict(bits=9), "quant bits must be in [1,8]"),
    (dict(group_size=0), "group_size must be >= 1"),
    (dict(rope_base=1.0), "rope: base must be > 1"),
    (dict(num_q_heads=12), "multiple of num_kv_heads"),
    (dict(batch=0), "must be positive"),
    (dict(head_dim=64), "head_dim == 128"),
    (dict(bits=4), "bits == 2"),
    (dict(max_tokens=0), "max_tokens"),
    (dict(num_kv_heads=128, num_q_heads=128, heads_per_group=4), "<= 8192"),
    (dict(num_kv_heads=64, num_q_heads=512, heads_per_group=64), "generic decode kernel's shared memory"),
])
def test_layer_validation_messages(lib, kw, msg):
    with pytest.raises(ValueError, match=re.escape(msg)):
        cfg(**kw).validate()


def test_every_power_of_two_rotation_is_accepted(lib):
    """RotationPlan::make accepts n = G*128 up to 2^13 with G | H
    (proj/src/hadamard.cpp:18-33); so does the layer (G = 8 .. 64 run on the
    generic kernels; GQA 4:1 at G = 4 on the tensor-core GQA kernel up to 8 KV
    heads, beyond on the generic one)."""
    for hkv, g, hq in ((8, 8, 8), (16, 16, 16), (64, 64, 64), (32, 32, 32), (16, 4, 64), (8, 4, 32), (64, 1, 64)):
        cfg(num_kv_heads=hkv, num_q_heads=hq, heads_per_group=g).validate()


def test_valid_configs(lib):
    for w_id in (1, 2, 3, 4, 5):
        from paper_2501_16383_b200.workload import CONFIGS

        w = CONFIGS[w_id]
        P.LayerConfig(batch=w.batch, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                      heads_per_group=w.heads_per_group, max_tokens=w.tokens + 1, rope_base=w.rope_base).validate()


def test_cache_bytes_and_carve(lib):
    c = cfg()
    d = c.desc()
    n = lib.rkv_cache_bytes(C.byref(d))
    C_ = 1024
    # codes 2*(B*T*C/16*4) + meta 2*(B*T*C/128*4) + sinks ... each 256-aligned
    assert n >= 2 * 2 * 64 * C_ // 4 + 2 * 2 * 64 * C_ // 32
    view = R.CacheView()
    buf = (C.c_uint8 * (n + 256))()
    base = (C.addressof(buf) + 255) // 256 * 256
    assert lib.rkv_cache_carve(C.byref(d), base, n, C.byref(view)) == 0
    ptrs = [getattr(view, f) for f, _ in R.CacheView._fields_]
    assert all(p % 256 == 0 for p in ptrs) and ptrs == sorted(ptrs)
    assert lib.rkv_cache_carve(C.byref(d), base, n - 1, C.byref(view)) == R.RKV_ERR_INVALID_ARGUMENT
    assert lib.rkv_cache_carve(C.byref(d), base + 16, n, C.byref(view)) == R.RKV_ERR_INVALID_ARGUMENT


def test_calibrate_reorder_host_matches_oracle(lib, oracle):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((64, 1024)).astype(np.float32)
    x[:, rng.integers(0, 1024, 10)] *= 30
    for stat in (P.STAT_SUM, P.STAT_MEAN_ABS):
        perm, inv = P.calibrate_reorder(x, stat)
        operm, oinv = oracle.calibrate_reorder(x, stat)
        assert np.array_equal(perm, operm) and np.array_equal(inv, oinv)
    # proj/tests/test_reorder.cpp:22-36 KATs through the ABI
    assert list(P.calibrate_reorder(np.float32([[3, -5, 1]]), P.STAT_SUM)[0]) == [1, 2, 0]
    assert list(P.calibrate_reorder(np.float32([[1, 1, 1, 1], [-1, -1, -1, -1]]), P.STAT_SUM)[0]) == [0, 1, 2, 3]
    with pytest.raises(ValueError, match="empty calibration set"):
        P.calibrate_reorder(np.zeros((0, 4), np.float32))


def test_detect_sinks_host_matches_oracle(lib, oracle):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 128, 512)).astype(np.float32)
    x[0, 0, 3] = 100.0
    x[1, 77, 9] = -120.0
    assert np.array_equal(P.detect_massive_activations(x), oracle.detect_sinks(x))
    assert np.flatnonzero(P.detect_massive_activations(x)).tolist() == [0, 77]
    with pytest.raises(ValueError, match="rel_threshold must be > 1"):
        P.detect_massive_activations(x, rel_threshold=1.0)


def test_apply_reorder_host_round_trip():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((3, 12)).astype(np.float32)
    perm = rng.permutation(12)
    y = P.apply_reorder(x, perm)
    assert np.array_equal(P.apply_reorder(y, perm, inverse=True), x)
    with pytest.raises(ValueError):
        P.apply_reorder(x, perm[:5])


def test_null_and_size_errors(lib):
    d = cfg().desc()
    assert lib.rkv_layer_validate(None) == R.RKV_ERR_INVALID_ARGUMENT
    assert lib.rkv_quantize_kv(C.byref(d), None, None, None, None, None, 0, None, None) == R.RKV_ERR_INVALID_ARGUMENT
    view = R.CacheView(*([256] * 9))
    # num_new == 0 is a no-op even without a GPU
    assert lib.rkv_quantize_kv(C.byref(d), None, None, None, None, None, 0, C.byref(view), None) == R.RKV_OK
    assert lib.rkv_quantize_kv(C.byref(d), None, None, None, None, None, -1, C.byref(view), None) == R.RKV_ERR_INVALID_ARGUMENT
    assert lib.rkv_decode_attention(C.byref(d), None, None, 0, C.byref(view), None, None, None, None, 0, None) \
        == R.RKV_ERR_INVALID_ARGUMENT
    assert b"null" in lib.rkv_last_error()


def test_fused_append_argument_errors(lib):
    """rkv_quantize_kv_fused validates before any device work (no GPU needed)."""
    d = cfg().desc()
    view = R.CacheView(*([256] * 9))
    f = lib.rkv_quantize_kv_fused
    assert f(C.byref(d), None, None, R.ROWS_F32, None, None, None, 0, None, None) == R.RKV_ERR_INVALID_ARGUMENT
    assert f(C.byref(d), None, None, R.ROWS_F32, None, None, None, 0, C.byref(view), None) == R.RKV_OK
    assert f(C.byref(d), None, None, 7, None, None, None, 0, C.byref(view), None) == R.RKV_ERR_INVALID_ARGUMENT
    assert b"dtype" in lib.rkv_last_error()
    assert f(C.byref(d), None, None, R.ROWS_F16, None, None, None, -1, C.byref(view), None) == R.RKV_ERR_INVALID_ARGUMENT
    assert f(C.byref(d), None, None, R.ROWS_F16, None, None, None, 4, C.byref(view), None) == R.RKV_ERR_INVALID_ARGUMENT
    assert b"non-null" in lib.rkv_last_error()
    raw = np.zeros(512, np.uint8)
    base = raw.ctypes.data + (-raw.ctypes.data) % 16  # 16-byte aligned
    buf, mis = C.c_void_p(base), C.c_void_p(base + 4)
    pos = (C.c_int64 * 4)()
    perm = (C.c_int32 * 4)()
    assert f(C.byref(d), mis, buf, R.ROWS_F32, perm, None, pos, 4, C.byref(view), None) == R.RKV_ERR_INVALID_ARGUMENT
    assert b"aligned" in lib.rkv_last_error()
    big = d.max_tokens + 1
    assert f(C.byref(d), buf, buf, R.ROWS_F32, perm, None, pos, big, C.byref(view), None) == R.RKV_ERR_OUT_OF_RANGE


def test_cpp_api_program_compiles(tmp_path, lib):
    """include/rotatekv/rotatekv.hpp + the C ABI link into a C++ program."""
    from tests._cpp import build_cpp_test

    assert os.path.exists(build_cpp_test(str(tmp_path)))
