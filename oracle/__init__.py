"""ctypes/numpy front end of the parity checkers (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  It wraps

* ``_build/librkv_oracle.so`` -- our C restatement (rkv_oracle.c), and
* ``_ref/librotatekv_ref.so`` -- the unmodified reference library compiled
  from /root/reference/proj/src by oracle/Makefile (optional: present when it
  was built in a container that had /root/reference).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "librkv_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librotatekv_ref.so")
REF_SRC = "/root/reference/proj"

SCALE_FP16_CEIL = 0
SCALE_E4M3_CEIL = 1
STAT_SUM = 0
STAT_MEAN_ABS = 1


def build(ref: bool = True) -> None:
    """Compile the restatement and (when the reference sources exist) _ref."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"REF={REF_SRC}"], check=True)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        _lib = C.CDLL(ORACLE_SO)
        L = _lib
        L.rkvo_half_to_float.restype = C.c_float
        L.rkvo_half_to_float.argtypes = [C.c_uint16]
        L.rkvo_float_to_half_rn.restype = C.c_uint16
        L.rkvo_float_to_half_rn.argtypes = [C.c_float]
        L.rkvo_fp16_ceil.restype = C.c_uint16
        L.rkvo_fp16_ceil.argtypes = [C.c_float]
        L.rkvo_e4m3_decode.restype = C.c_float
        L.rkvo_e4m3_decode.argtypes = [C.c_uint8]
        L.rkvo_e4m3_encode.restype = C.c_uint8
        L.rkvo_e4m3_encode.argtypes = [C.c_float]
        L.rkvo_e4m3_encode_ceil.restype = C.c_uint8
        L.rkvo_e4m3_encode_ceil.argtypes = [C.c_float]
        L.rkvo_fwht_inplace.argtypes = [C.c_void_p, C.c_int64]
        L.rkvo_rotate_rows.argtypes = [C.c_void_p] + [C.c_int64] * 4
        L.rkvo_apply_reorder.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int, C.c_void_p]
        L.rkvo_invert_perm.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.rkvo_calibrate_reorder.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        L.rkvo_apply_rope_rows.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_void_p, C.c_int]
        L.rkvo_pack_codes.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        L.rkvo_unpack_codes.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        L.rkvo_quantize_group.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.rkvo_dequantize_group.argtypes = [C.c_void_p, C.c_int64, C.c_float, C.c_uint8, C.c_void_p]
        L.rkvo_quantize_kv_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int] + [C.c_void_p] * 4
        L.rkvo_decode_attention.argtypes = [C.c_void_p] * 7 + [C.c_int64, C.c_void_p] + [C.c_int64] * 4 + [C.c_void_p, C.c_double, C.c_void_p]
        L.rkvo_detect_sinks.restype = C.c_int64
        L.rkvo_detect_sinks.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_void_p]
    return _lib


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The unmodified reference library (raises if it was never built)."""
    global _ref
    if _ref is None:
        if not have_ref():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        _ref = C.CDLL(REF_SO)
        R = _ref
        R.ref_fwht.argtypes = [C.c_void_p, C.c_int64]
        R.ref_rotate_rows.argtypes = [C.c_void_p] + [C.c_int64] * 4
        R.ref_apply_reorder.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int, C.c_void_p]
        R.ref_calibrate_reorder.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        R.ref_e4m3_decode.restype = C.c_float
        R.ref_e4m3_decode.argtypes = [C.c_uint8]
        R.ref_e4m3_encode.restype = C.c_uint8
        R.ref_e4m3_encode.argtypes = [C.c_float]
        R.ref_e4m3_encode_ceil.restype = C.c_uint8
        R.ref_e4m3_encode_ceil.argtypes = [C.c_float]
        R.ref_quantize_group.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int64] + [C.c_void_p] * 4
        R.ref_apply_rope_rows.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_void_p, C.c_int]
        R.ref_detect_sinks.restype = C.c_int64
        R.ref_detect_sinks.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_void_p]
        R.ref_prefill.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                  C.c_double, C.c_void_p]
        R.ref_cache_serialize.restype = C.c_int64
        R.ref_cache_serialize.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 4 + [C.c_void_p] * 2 + [C.c_int64]
        R.ref_cache_reserialize.restype = C.c_int64
        R.ref_cache_reserialize.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
        R.ref_quantize_kv_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p] + [C.c_void_p] * 6
        R.ref_decode_step.argtypes = [C.c_int64] * 3 + [C.c_void_p] * 3 + [C.c_int64, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
        R.ref_bench_create.restype = C.c_void_p
        R.ref_bench_create.argtypes = [C.c_int64] * 5 + [C.c_void_p, C.c_double, C.c_uint64, C.c_int]
        R.ref_bench_step.restype = C.c_double
        R.ref_bench_step.argtypes = [C.c_void_p, C.c_int]
        R.ref_bench_destroy.argtypes = [C.c_void_p]
        R.ref_bench_set_memo.argtypes = [C.c_void_p, C.c_int]
        R.ref_cache_rows.argtypes = [C.c_int64] * 3 + [C.c_void_p] * 3 + [C.c_int64] + [C.c_void_p] * 3
        R.ref_decode_step_routed.argtypes = ([C.c_int64] * 3 + [C.c_void_p] * 3 + [C.c_int64, C.c_void_p, C.c_int64,
                                             C.c_void_p, C.c_double, C.c_void_p, C.c_void_p])
    return _ref


# ----------------------------------------------------------------- wrappers

def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def fwht(v, impl="oracle"):
    v = f32(v).copy()
    rc = (lib().rkvo_fwht_inplace if impl == "oracle" else ref().ref_fwht)(_p(v), v.size)
    if rc != 0:
        raise ValueError("fwht: length must be a power of two")
    return v


def rotate_rows(x, head_dim, heads_per_group, num_heads, impl="oracle"):
    x = f32(x).copy()
    rows = x.size // (head_dim * num_heads)
    fn = lib().rkvo_rotate_rows if impl == "oracle" else ref().ref_rotate_rows
    if fn(_p(x), rows, head_dim, heads_per_group, num_heads) != 0:
        raise ValueError("rotate_rows: invalid rotation plan")
    return x


def apply_reorder(x, perm, inverse=False, impl="oracle"):
    x = f32(x)
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    c = perm.size
    out = np.empty_like(x)
    fn = lib().rkvo_apply_reorder if impl == "oracle" else ref().ref_apply_reorder
    if fn(_p(x), x.size // c, c, _p(perm), int(inverse), _p(out)) != 0:
        raise ValueError("apply_reorder failed")
    return out


def calibrate_reorder(rows, stat=STAT_SUM, impl="oracle"):
    rows = f32(rows)
    n, c = rows.shape
    perm = np.empty(c, np.int32)
    inv = np.empty(c, np.int32)
    if impl == "oracle":
        rc = lib().rkvo_calibrate_reorder(_p(rows), n, c, stat, _p(perm), _p(inv))
    else:
        assert stat == STAT_SUM
        rc = ref().ref_calibrate_reorder(_p(rows), n, c, _p(perm), _p(inv))
    if rc != 0:
        raise ValueError("calibrate_reorder failed")
    return perm, inv


def apply_rope_rows(x, num_heads, head_dim, base, positions, inverse=False, impl="oracle"):
    x = f32(x).copy()
    positions = np.ascontiguousarray(positions, dtype=np.int64)
    fn = lib().rkvo_apply_rope_rows if impl == "oracle" else ref().ref_apply_rope_rows
    if fn(_p(x), positions.size, num_heads, head_dim, float(base), _p(positions), int(inverse)) != 0:
        raise ValueError("rope failed")
    return x


def quantize_group(x, bits=2, scale_format=SCALE_FP16_CEIL):
    x = f32(x)
    codes = np.empty(x.size, np.uint8)
    s = C.c_float()
    z = C.c_uint8()
    sc = C.c_uint16()
    if lib().rkvo_quantize_group(_p(x), x.size, bits, scale_format, C.byref(s), C.byref(z), _p(codes), C.byref(sc)) != 0:
        raise ValueError("quantize_group failed")
    return s.value, z.value, codes, sc.value


def ref_quantize_group(x, bits=2, group_size=128):
    x = f32(x)
    codes = np.empty(x.size, np.uint8)
    packed = np.empty((x.size * bits + 7) // 8, np.uint8)
    sc = C.c_uint8()
    z = C.c_uint8()
    if ref().ref_quantize_group(_p(x), x.size, bits, group_size, _p(codes), _p(packed), C.byref(sc), C.byref(z)) != 0:
        raise ValueError("ref quantize_group failed")
    return sc.value, z.value, codes, packed


def pack_codes(codes, bits):
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    out = np.empty((codes.size * bits + 7) // 8, np.uint8)
    lib().rkvo_pack_codes(_p(codes), codes.size, bits, _p(out))
    return out


def unpack_codes(packed, n, bits):
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    out = np.empty(n, np.uint8)
    lib().rkvo_unpack_codes(_p(packed), n, bits, _p(out))
    return out


def quantize_kv_rows(k_raw, v_raw, num_kv_heads, head_dim, heads_per_group, perm,
                     scale_format=SCALE_FP16_CEIL):
    """k_raw/v_raw: uint16 fp16 bits or float16 [rows, C]."""
    k_raw = np.ascontiguousarray(k_raw).view(np.uint16)
    v_raw = np.ascontiguousarray(v_raw).view(np.uint16)
    rows, c = k_raw.shape
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    kc = np.empty((rows, c // 16), np.uint32)
    km = np.empty((rows, c // 128), np.uint32)
    vc = np.empty((rows, c // 16), np.uint32)
    vm = np.empty((rows, c // 128), np.uint32)
    rc = lib().rkvo_quantize_kv_rows(_p(k_raw), _p(v_raw), rows, num_kv_heads, head_dim,
                                     heads_per_group, _p(perm), scale_format, _p(kc), _p(km), _p(vc), _p(vm))
    if rc != 0:
        raise ValueError("quantize_kv_rows failed")
    return kc, km, vc, vm


def ref_quantize_kv_rows(k, v, num_heads, head_dim, heads_per_group, perm):
    """Unmodified reference chain (e4m3 scales).  k, v: float32 [rows, C]."""
    k = f32(k)
    v = f32(v)
    rows, c = k.shape
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    kc = np.empty((rows, c // 16), np.uint32)
    vc = np.empty((rows, c // 16), np.uint32)
    ks = np.empty((rows, c // 128), np.uint8)
    kz = np.empty((rows, c // 128), np.uint8)
    vs = np.empty((rows, c // 128), np.uint8)
    vz = np.empty((rows, c // 128), np.uint8)
    rc = ref().ref_quantize_kv_rows(_p(k), _p(v), rows, num_heads, head_dim, heads_per_group,
                                    _p(perm), _p(kc), _p(ks), _p(kz), _p(vc), _p(vs), _p(vz))
    if rc != 0:
        raise ValueError("ref_quantize_kv_rows failed")
    return kc, ks, kz, vc, vs, vz


def decode_attention(k_codes, k_meta, v_codes, v_meta, is_sink, sink_k, sink_v, q,
                     num_q_heads, num_kv_heads, head_dim, heads_per_group, perm, rope_base):
    """One sequence.  codes/meta: [T, ...] u32; sink_k/sink_v: fp16 [T, C]
    (rows used only where is_sink); q: fp16 [Hq*d].  Returns fp32 [Hq, d]."""
    T = k_codes.shape[0]
    c = num_kv_heads * head_dim
    arrs = [np.ascontiguousarray(a) for a in (k_codes, k_meta, v_codes, v_meta)]
    is_sink = np.ascontiguousarray(is_sink, dtype=np.uint8)
    sk = np.ascontiguousarray(sink_k).view(np.uint16).reshape(T, c)
    sv = np.ascontiguousarray(sink_v).view(np.uint16).reshape(T, c)
    q = np.ascontiguousarray(q).view(np.uint16).reshape(-1)
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    out = np.empty((num_q_heads, head_dim), np.float32)
    rc = lib().rkvo_decode_attention(*[_p(a) for a in arrs], _p(is_sink), _p(sk), _p(sv), T, _p(q),
                                     num_q_heads, num_kv_heads, head_dim, heads_per_group, _p(perm),
                                     float(rope_base), _p(out))
    if rc != 0:
        raise ValueError("decode_attention failed")
    return out


def ref_prefill(x, sink, perm, num_heads, head_dim, heads_per_group, rope_base):
    """The reference's prefill attention output [T, C] (identity projections:
    x rows are keys, values and queries; token 0 + flagged tokens are sinks)."""
    x = f32(x)
    sink = np.ascontiguousarray(sink, np.uint8)
    perm = np.ascontiguousarray(perm, np.int32)
    out = np.empty_like(x)
    if ref().ref_prefill(num_heads, head_dim, heads_per_group, _p(x), _p(sink), x.shape[0], _p(perm),
                         float(rope_base), _p(out)) != 0:
        raise ValueError("ref_prefill failed")
    return out


def ref_cache_serialize(k_raw, v_raw, sink, perm, num_heads, head_dim, heads_per_group):
    """The reference's LayerKVCache::serialize of raw rows appended as prefill does."""
    k, v = f32(k_raw), f32(v_raw)
    sink = np.ascontiguousarray(sink, np.uint8)
    perm = np.ascontiguousarray(perm, np.int32)
    rows = k.shape[0]
    n = ref().ref_cache_serialize(_p(k), _p(v), _p(sink), rows, num_heads, head_dim, heads_per_group, _p(perm),
                                  None, 0)
    if n < 0:
        raise ValueError("ref_cache_serialize failed")
    out = np.empty(n, np.uint8)
    ref().ref_cache_serialize(_p(k), _p(v), _p(sink), rows, num_heads, head_dim, heads_per_group, _p(perm),
                              _p(out), n)
    return out.tobytes()


def ref_cache_reserialize(data):
    """LayerKVCache::deserialize + serialize in the reference (None if it throws)."""
    buf = np.frombuffer(data, np.uint8).copy()
    n = ref().ref_cache_reserialize(_p(buf), buf.size, None, 0)
    if n < 0:
        return None
    out = np.empty(n, np.uint8)
    ref().ref_cache_reserialize(_p(buf), buf.size, _p(out), n)
    return out.tobytes()


def ref_decode_step(k_raw, v_raw, sink, perm, x, num_heads, head_dim, heads_per_group, rope_base):
    k_raw = f32(k_raw)
    v_raw = f32(v_raw)
    T, c = k_raw.shape
    sink = np.ascontiguousarray(sink, dtype=np.uint8)
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    x = f32(x)
    out = np.empty(c, np.float32)
    rc = ref().ref_decode_step(num_heads, head_dim, heads_per_group, _p(k_raw), _p(v_raw), _p(sink), T,
                               _p(perm), float(rope_base), _p(x), _p(out))
    if rc != 0:
        raise ValueError("ref_decode_step failed")
    return out


def ref_cache_rows(k_raw, v_raw, sink, perm, num_heads, head_dim, heads_per_group):
    """The reference's LayerKVCache::keys()/values() after appending the rows
    (fused frame; e4m3 scales)."""
    k_raw = f32(k_raw)
    v_raw = f32(v_raw)
    T, c = k_raw.shape
    sink = np.ascontiguousarray(sink, dtype=np.uint8)
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    ko = np.empty((T, c), np.float32)
    vo = np.empty((T, c), np.float32)
    if ref().ref_cache_rows(num_heads, head_dim, heads_per_group, _p(k_raw), _p(v_raw), _p(sink), T, _p(perm), _p(ko),
                            _p(vo)) != 0:
        raise ValueError("ref_cache_rows failed")
    return ko, vo


def ref_decode_step_routed(k_raw, v_raw, sink, promote, perm, x, num_heads, head_dim, heads_per_group, rope_base):
    """The reference's cache filled with append-time sinks `sink`, then
    route_sinks(promote) with the fused-frame rows, then one decode_step."""
    k_raw = f32(k_raw)
    v_raw = f32(v_raw)
    T, c = k_raw.shape
    sink = np.ascontiguousarray(sink, dtype=np.uint8)
    promote = np.ascontiguousarray(promote, dtype=np.int64)
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    x = f32(x)
    out = np.empty(c, np.float32)
    rc = ref().ref_decode_step_routed(num_heads, head_dim, heads_per_group, _p(k_raw), _p(v_raw), _p(sink), T,
                                      _p(promote), promote.size, _p(perm), float(rope_base), _p(x), _p(out))
    if rc == -1:
        raise IndexError("ref_decode_step_routed: the reference threw")
    if rc != 0:
        raise ValueError(f"ref_decode_step_routed failed ({rc})")
    return out


def detect_sinks(hidden, rel=50.0, abs_floor=0.0, impl="oracle"):
    hidden = f32(hidden)
    b, s, h = hidden.shape
    flags = np.empty(s, np.uint8)
    fn = lib().rkvo_detect_sinks if impl == "oracle" else ref().ref_detect_sinks
    n = fn(_p(hidden), b, s, h, float(rel), float(abs_floor), _p(flags))
    if n < 0:
        raise ValueError("detect_sinks failed")
    return flags


def half_to_float(h):
    return lib().rkvo_half_to_float(int(h))


def float_to_half(f):
    return lib().rkvo_float_to_half_rn(float(f))


def fp16_ceil(f):
    return lib().rkvo_fp16_ceil(float(f))


def e4m3_decode(c, impl="oracle"):
    return (lib().rkvo_e4m3_decode if impl == "oracle" else ref().ref_e4m3_decode)(int(c))


def e4m3_encode(x, impl="oracle"):
    return (lib().rkvo_e4m3_encode if impl == "oracle" else ref().ref_e4m3_encode)(float(x))


def e4m3_encode_ceil(x, impl="oracle"):
    return (lib().rkvo_e4m3_encode_ceil if impl == "oracle" else ref().ref_e4m3_encode_ceil)(float(x))
