"""Python host layer over the C ABI (include/rotatekv/rotatekv.h).

Mirrors the reference's hot-path API (namespace rotatekv,
/root/reference/proj/include/rotatekv/*.hpp) with the same names, argument
meaning and error classes:

    reference (C++)                           here
    ----------------------------------------  -------------------------------------------
    calibrate_reorder(rotated keys)           calibrate_reorder(rows, stat)
    apply_reorder(x, plan, layer, inverse)    apply_reorder(x, perm, inverse)
    rotate_rows(x, plan, inverse)             rotate_keys(layer, k)          (device FWHT)
    detect_massive_activations(block, rel)    detect_massive_activations(hidden, rel, floor)
    LayerKVCache(cfg, C) + append(k, v, sink) RotateKVLayer(...).append(k, v, sink_flags)
    decode_step attention half                RotateKVLayer.decode(q)  /  .decode_step(k, v, q)

std::invalid_argument -> ValueError, std::out_of_range -> IndexError,
std::runtime_error -> RuntimeError.  Device tensors are torch CUDA tensors;
torch is only the allocator/stream provider.  There is no CPU fallback: if
the sm_100a library is missing the import of the device path fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RKV_LIB") or os.path.join(_PKG, "_lib", "librotatekv_b200.so")  # RKV_LIB: A/B builds

RKV_OK, RKV_ERR_INVALID_ARGUMENT, RKV_ERR_OUT_OF_RANGE, RKV_ERR_RUNTIME, RKV_ERR_CUDA = range(5)
SCALE_FP16_CEIL, SCALE_E4M3_CEIL = 0, 1
ROWS_F32, ROWS_F16 = 0, 1  # rkv_rows_dtype: fused-frame append inputs
STAT_SUM, STAT_MEAN_ABS = 0, 1


class LayerDesc(C.Structure):
    _fields_ = [
        ("batch", C.c_int32),
        ("num_q_heads", C.c_int32),
        ("num_kv_heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("heads_per_group", C.c_int32),
        ("group_size", C.c_int32),
        ("bits", C.c_int32),
        ("scale_format", C.c_int32),
        ("max_tokens", C.c_int64),
        ("max_sinks", C.c_int32),
        ("reserved", C.c_int32),
        ("rope_base", C.c_double),
    ]


class CacheView(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "k_codes", "v_codes", "k_meta", "v_meta", "sink_k", "sink_v", "sink_pos", "sink_count", "sink_mask")]


_lib = None


def lib():
    """Load the sm_100a C-ABI library; raises if it was never built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2501_16383_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        D = C.POINTER(LayerDesc)
        L.rkv_last_error.restype = C.c_char_p
        L.rkv_version.restype = C.c_char_p
        L.rkv_layer_validate.argtypes = [D]
        L.rkv_cache_bytes.restype = C.c_size_t
        L.rkv_cache_bytes.argtypes = [D]
        L.rkv_cache_carve.argtypes = [D, P, C.c_size_t, C.POINTER(CacheView)]
        L.rkv_cache_reset.argtypes = [D, C.POINTER(CacheView), P]
        L.rkv_rope_table_bytes.restype = C.c_size_t
        L.rkv_rope_table_bytes.argtypes = [D, C.c_int64]
        L.rkv_rope_table_init.argtypes = [D, P, C.c_int64, P]
        L.rkv_quantize_kv.argtypes = [D, P, P, P, P, P, C.c_int64, C.POINTER(CacheView), P]
        L.rkv_quantize_kv_fused.argtypes = [D, P, P, C.c_int32, P, P, P, C.c_int64, C.POINTER(CacheView), P]
        L.rkv_decode_workspace_bytes.restype = C.c_size_t
        L.rkv_decode_workspace_bytes.argtypes = [D, C.c_int64]
        L.rkv_decode_attention.argtypes = [D, P, P, C.c_int64, C.POINTER(CacheView), P, P, P, P, C.c_size_t, P]
        L.rkv_decode_attention_partial.argtypes = [D, P, P, P, P, C.c_int64, C.POINTER(CacheView), P, P, P, P, P,
                                                   C.c_size_t, P]
        L.rkv_decode_merge.argtypes = [D, P, P, C.c_int32, P, P, C.POINTER(CacheView), P, P, P]
        L.rkv_layer_plan_bytes.restype = C.c_size_t
        L.rkv_layer_plan_bytes.argtypes = [D]
        L.rkv_layer_plan_build.argtypes = [D, P, P, C.c_size_t, C.POINTER(C.c_int32)]
        L.rkv_layer_plan_init.argtypes = [D, P, P, C.c_size_t, P]
        L.rkv_rotate_keys.argtypes = [D, P, C.c_int64, P, P]
        L.rkv_calibrate_reorder.argtypes = [P, C.c_int64, C.c_int64, C.c_int32, P, P]
        L.rkv_detect_sinks.argtypes = [P, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, P,
                                       C.POINTER(C.c_int64)]
        L.rkv_detect_sinks_workspace_bytes.restype = C.c_size_t
        L.rkv_detect_sinks_workspace_bytes.argtypes = []
        L.rkv_detect_sinks_device.argtypes = [P, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, P, P, P,
                                              C.c_size_t, P]
        L.rkv_prefill_workspace_bytes.restype = C.c_size_t
        L.rkv_prefill_workspace_bytes.argtypes = [D, C.c_int64, C.c_int64]
        L.rkv_prefill_attention.argtypes = [D, P, C.c_int64, P, P, C.c_int64, P, P, P, P, P, C.c_size_t, P]
        L.rkv_cache_wire_bytes.restype = C.c_size_t
        L.rkv_cache_wire_bytes.argtypes = [D, C.c_int64, C.c_int64, C.c_int32]
        L.rkv_cache_export.argtypes = [D, P, C.c_int64, C.c_int64, P, C.c_int32, P, C.c_size_t, P, P]
        L.rkv_cache_import.argtypes = [D, P, C.c_size_t, P, C.c_int64, P, P, P]
        L.rkv_calibrate_workspace_bytes.restype = C.c_size_t
        L.rkv_calibrate_workspace_bytes.argtypes = [D, C.c_int64]
        L.rkv_calibrate_reorder_device.argtypes = [D, P, C.c_int64, C.c_int32, P, C.c_size_t, P, P, P]
        L.rkv_promote_sinks.argtypes = [D, C.POINTER(CacheView), P, C.c_int64, P, P, P, P]
        L.rkv_cache_read.argtypes = [D, C.POINTER(CacheView), P, C.c_int64, C.c_int64, C.c_int64, C.c_int32, P, P, P]
        L.rkv_set_debug_option.argtypes = [C.c_char_p, C.c_int64]
        L.rkv_decode_plan_info.argtypes = [D, C.c_int64, C.POINTER(C.c_int64)]
        for name in ("rkv_promote_sinks", "rkv_set_debug_option", "rkv_decode_plan_info", "rkv_cache_read", "rkv_layer_validate", "rkv_cache_carve", "rkv_cache_reset", "rkv_rope_table_init",
                     "rkv_quantize_kv", "rkv_quantize_kv_fused", "rkv_decode_attention", "rkv_rotate_keys", "rkv_calibrate_reorder",
                     "rkv_detect_sinks", "rkv_detect_sinks_device", "rkv_layer_plan_build", "rkv_layer_plan_init",
                     "rkv_calibrate_reorder_device", "rkv_cache_export", "rkv_cache_import",
                     "rkv_prefill_attention", "rkv_decode_attention_partial", "rkv_decode_merge"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status == RKV_OK:
        return
    msg = lib().rkv_last_error().decode()
    if status == RKV_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == RKV_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


def _ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def _np(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


@dataclass
class LayerConfig:
    """One attention layer (PipelineConfig + QuantConfig + RotationPlan)."""
    batch: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int = 128
    heads_per_group: int = 4
    max_tokens: int = 4096
    max_sinks: int = 8
    rope_base: float = 10000.0
    scale_format: int = SCALE_FP16_CEIL
    group_size: int = 128
    bits: int = 2

    def desc(self) -> LayerDesc:
        return LayerDesc(self.batch, self.num_q_heads, self.num_kv_heads, self.head_dim, self.heads_per_group,
                         self.group_size, self.bits, self.scale_format, self.max_tokens, self.max_sinks, 0,
                         float(self.rope_base))

    @property
    def channels(self) -> int:
        return self.num_kv_heads * self.head_dim

    def validate(self) -> None:
        d = self.desc()
        _check(lib().rkv_layer_validate(C.byref(d)))


# ------------------------------------------------------------ host helpers

def set_debug_option(name: str, value: int) -> None:
    """Process-global experiment switch (rkv_set_debug_option): kernel
    selection etc.  Build layers (plan + RoPE table) after changing one."""
    _check(lib().rkv_set_debug_option(name.encode(), int(value)))


def decode_plan_info(cfg, max_seq_len: int) -> dict:
    """The decode plan rkv_decode_attention uses for this layer shape
    (diagnostic, rkv_decode_plan_info)."""
    out = (C.c_int64 * 10)()
    d = cfg.desc()
    _check(lib().rkv_decode_plan_info(C.byref(d), int(max_seq_len), out))
    keys = ("kind", "tile_channels", "threads", "splits", "partials", "chunk", "tile_tokens", "ctas_per_sm",
            "smem", "stages")
    return dict(zip(keys, [int(x) for x in out]))


WIRE_REFERENCE, WIRE_FP16_SCALE = 0, 1


def calibrate_reorder(rotated_keys, stat: int = STAT_MEAN_ABS):
    """calibrate_reorder (proj/src/reorder.cpp:91-110) -> (perm, inverse) int32.
    rotated_keys: [rows, C] float (host).  stat: STAT_SUM (reference) or
    STAT_MEAN_ABS (north star)."""
    x = _np(rotated_keys, np.float32)
    if x.ndim != 2:
        raise ValueError("expected [b,h,s,d] or [tokens, channels]")
    perm = np.empty(x.shape[1], np.int32)
    inv = np.empty(x.shape[1], np.int32)
    _check(lib().rkv_calibrate_reorder(x.ctypes.data, x.shape[0], x.shape[1], stat, perm.ctypes.data,
                                       inv.ctypes.data))
    return perm, inv


def apply_reorder(x, perm, inverse: bool = False):
    """apply_reorder (proj/src/reorder.cpp:112-128): dst[j] = src[p[j]]."""
    perm = np.asarray(perm)
    if x.shape[-1] != perm.size:
        raise ValueError("apply_reorder: trailing dimension mismatch")
    if inverse:
        inv = np.empty_like(perm)
        inv[perm] = np.arange(perm.size, dtype=perm.dtype)
        perm = inv
    return x[..., perm]


def detect_massive_activations(hidden, rel_threshold: float = 50.0, abs_floor: float = 0.0):
    """detect_massive_activations (proj/src/sink.cpp:14-45) -> uint8 flags [s]."""
    h = _np(hidden, np.float32)
    if h.ndim != 3:
        raise ValueError("detect_massive_activations: expected [b,s,hidden]")
    flags = np.empty(h.shape[1], np.uint8)
    n = C.c_int64()
    _check(lib().rkv_detect_sinks(h.ctypes.data, h.shape[0], h.shape[1], h.shape[2], float(rel_threshold),
                                  float(abs_floor), flags.ctypes.data, C.byref(n)))
    return flags


def detect_massive_activations_device(hidden, rel_threshold: float = 50.0, abs_floor: float = 0.0,
                                     return_median: bool = False):
    """detect_massive_activations on the GPU: hidden = CUDA fp32 [b, s, h]
    tensor -> CUDA uint8 flags [s] (and the median of |hidden|), no host
    round trip; the flags feed RotateKVLayer.append_device after a broadcast
    over the batch."""
    torch = __import__("torch")
    if hidden.ndim != 3:
        raise ValueError("detect_massive_activations: expected [b,s,hidden]")
    if hidden.dtype != torch.float32 or not hidden.is_cuda:
        raise ValueError("detect_massive_activations: hidden must be a CUDA float32 tensor")
    hidden = hidden.contiguous()
    b, s_, h = hidden.shape
    flags = torch.empty(s_, dtype=torch.uint8, device=hidden.device)
    median = torch.empty(1, dtype=torch.float32, device=hidden.device)
    nws = lib().rkv_detect_sinks_workspace_bytes()
    ws = torch.empty(nws, dtype=torch.uint8, device=hidden.device)
    stream = C.c_void_p(torch.cuda.current_stream(hidden.device).cuda_stream)
    _check(lib().rkv_detect_sinks_device(_ptr(hidden), b, s_, h, float(rel_threshold), float(abs_floor), _ptr(flags),
                                         _ptr(median), _ptr(ws), nws, stream))
    return (flags, median) if return_median else flags


def layer_plan_build(cfg: LayerConfig, perm):
    """Host build of the decode plan (scatter word assignment) -> (uint32
    words, cost = summed worst bank-slot multiplicity, 16 per half-warp ideal)."""
    d = cfg.desc()
    perm = _np(perm, np.int32)
    n = lib().rkv_layer_plan_bytes(C.byref(d))
    out = np.zeros(n // 4, np.uint32)
    cost = C.c_int32()
    _check(lib().rkv_layer_plan_build(C.byref(d), perm.ctypes.data, out.ctypes.data, n, C.byref(cost)))
    return out, cost.value


# ------------------------------------------------------------ device layer

class RotateKVLayer:
    """One layer's 2-bit rotated KV cache on a CUDA device.

    Host-side mirrors of every sequence's length and sink count give the
    reference's argument checks (position == cache length, out-of-range
    tokens, sidecar capacity) without a device round trip."""

    def __init__(self, cfg: LayerConfig, perm, device="cuda", stream=None):
        import torch

        self.torch = torch
        self.cfg = cfg
        cfg.validate()
        self.device = torch.device(device)
        self._desc = cfg.desc()
        c = cfg.channels
        perm = _np(perm, np.int32)
        if perm.shape != (c,) or not np.array_equal(np.sort(perm), np.arange(c)):
            raise ValueError("reorder plan: perm must be a permutation of the channel count")
        self.perm_host = perm
        self.perm = torch.from_numpy(perm).to(self.device)
        nbytes = lib().rkv_cache_bytes(C.byref(self._desc))
        self._buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = (self._buf.data_ptr() + 255) // 256 * 256
        self._view = CacheView()
        _check(lib().rkv_cache_carve(C.byref(self._desc), base, nbytes, C.byref(self._view)))
        self._base = base
        rope_bytes = lib().rkv_rope_table_bytes(C.byref(self._desc), cfg.max_tokens)
        self.rope = torch.empty(rope_bytes // 4, dtype=torch.float32, device=self.device)
        plan_bytes = lib().rkv_layer_plan_bytes(C.byref(self._desc))
        self.plan = torch.empty(plan_bytes, dtype=torch.uint8, device=self.device)
        _check(lib().rkv_layer_plan_init(C.byref(self._desc), perm.ctypes.data, _ptr(self.plan), plan_bytes,
                                         self._stream_or_none(stream)))
        self.lengths = np.zeros(cfg.batch, np.int64)
        self.sink_counts = np.zeros(cfg.batch, np.int64)
        self.sink_tokens = [set() for _ in range(cfg.batch)]  # host mirror of the sink masks
        self._ws = None
        self._ws_for = None
        self.stream = stream
        _check(lib().rkv_rope_table_init(C.byref(self._desc), _ptr(self.rope), cfg.max_tokens, self._stream()))
        self.reset()

    # -- plumbing
    def _stream_or_none(self, stream):
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        return C.c_void_p(s.cuda_stream)

    def _stream(self):
        s = self.stream if self.stream is not None else self.torch.cuda.current_stream(self.device)
        return C.c_void_p(s.cuda_stream)

    def reset(self):
        _check(lib().rkv_cache_reset(C.byref(self._desc), C.byref(self._view), self._stream()))
        self.lengths[:] = 0
        self.sink_counts[:] = 0
        self.sink_tokens = [set() for _ in range(self.cfg.batch)]

    def _arr(self, name, dtype, shape):
        """A torch view of one carved cache array."""
        torch = self.torch
        off = getattr(self._view, name) - self._base
        n = int(np.prod(shape))
        esz = torch.empty((), dtype=dtype).element_size()
        start = (self._base - self._buf.data_ptr()) + off
        return self._buf[start:start + n * esz].view(dtype).view(*shape)

    def arrays(self):
        """Device views: k_codes/v_codes [B,T,C/16] int32 (u32 bits), k_meta/v_meta
        [B,T,C/128] int32, sink_k/sink_v [B,S,C] fp16, sink_pos [B,S], sink_count [B],
        sink_mask [B,ceil(T/32)]."""
        t = self.torch
        B, T, S, Cc = self.cfg.batch, self.cfg.max_tokens, self.cfg.max_sinks, self.cfg.channels
        return {
            "k_codes": self._arr("k_codes", t.int32, (B, T, Cc // 16)),
            "v_codes": self._arr("v_codes", t.int32, (B, T, Cc // 16)),
            "k_meta": self._arr("k_meta", t.int32, (B, T, Cc // 128)),
            "v_meta": self._arr("v_meta", t.int32, (B, T, Cc // 128)),
            "sink_k": self._arr("sink_k", t.float16, (B, max(S, 1), Cc)),
            "sink_v": self._arr("sink_v", t.float16, (B, max(S, 1), Cc)),
            "sink_pos": self._arr("sink_pos", t.int32, (B, max(S, 1))),
            "sink_count": self._arr("sink_count", t.int32, (B,)),
            "sink_mask": self._arr("sink_mask", t.int32, (B, (T + 31) // 32)),
        }

    # -- the attention half of prefill (proj/src/pipeline.cpp:156-191): causal, over the cache
    def prefill_attention(self, q, q_start=None, out=None):
        """q: [B, nq, Hq, 128] fp16 pre-RoPE; row i of sequence b is the query at
        position q_start[b] + i (default: the last nq cached tokens) and attends
        causally to cache tokens 0 .. that position.  Returns fp32 [B, nq, Hq, 128]
        with V's rotation undone."""
        torch = self.torch
        B, Hq = self.cfg.batch, self.cfg.num_q_heads
        if q.dtype != torch.float16 or q.dim() != 4 or q.shape[0] != B or q.shape[2] != Hq or q.shape[3] != 128:
            raise ValueError("prefill: q must be [batch, num_q, Hq, 128] fp16")
        nq = q.shape[1]
        start = self.lengths - nq if q_start is None else _np(q_start, np.int64)
        if np.any(start < 0) or np.any(start + nq > self.lengths):
            raise IndexError("prefill: query positions must lie inside the cache")
        q = q.contiguous()
        if out is None:
            out = torch.empty(B, nq, Hq, 128, dtype=torch.float32, device=self.device)
        mx = int(self.lengths.max())
        nws = lib().rkv_prefill_workspace_bytes(C.byref(self._desc), nq, mx)
        ws = torch.empty(max(nws, 1), dtype=torch.uint8, device=self.device)
        st = torch.from_numpy(np.ascontiguousarray(start)).to(self.device)
        ln = torch.from_numpy(self.lengths.copy()).to(self.device)
        _check(lib().rkv_prefill_attention(C.byref(self._desc), _ptr(q), nq, _ptr(st), _ptr(ln), mx,
                                           C.byref(self._view), _ptr(self.plan), _ptr(self.rope), _ptr(out),
                                           _ptr(ws), nws, self._stream()))
        return out

    # -- LayerKVCache::serialize / deserialize (proj/src/kv_cache.cpp:119-173), one sequence
    def serialize(self, seq: int, fmt: int = None) -> bytes:
        """Wire bytes of sequence `seq` (its current length).  fmt:
        WIRE_REFERENCE (the reference's byte format, e4m3 scales) or
        WIRE_FP16_SCALE; default: the one matching the layer's scale_format."""
        if fmt is None:
            fmt = WIRE_REFERENCE if self.cfg.scale_format == SCALE_E4M3_CEIL else WIRE_FP16_SCALE
        n = int(self.lengths[seq]) if 0 <= seq < self.cfg.batch else 0  # the C ABI reports a bad index
        cap = lib().rkv_cache_wire_bytes(C.byref(self._desc), n, min(n, self.cfg.max_sinks), fmt)  # upper bound
        out = np.empty(max(cap, 1), np.uint8)
        written = C.c_size_t()
        _check(lib().rkv_cache_export(C.byref(self._desc), C.byref(self._view), seq, n, self.perm_host.ctypes.data,
                                      fmt, out.ctypes.data, out.size, C.byref(written), self._stream()))
        return out[:written.value].tobytes()

    def deserialize(self, data: bytes, seq: int) -> int:
        """Replace sequence `seq` with the serialized cache; returns its token count."""
        buf = np.frombuffer(data, np.uint8)
        n = C.c_int64()
        _check(lib().rkv_cache_import(C.byref(self._desc), buf.ctypes.data if buf.size else None, buf.size,
                                      self.perm_host.ctypes.data, seq, C.byref(self._view), C.byref(n),
                                      self._stream()))
        self.lengths[seq] = n.value
        self.sink_counts[seq] = int(self.arrays()["sink_count"][seq].item())
        cnt = int(self.sink_counts[seq])
        self.sink_tokens[seq] = set(int(t) for t in self.arrays()["sink_pos"][seq, :cnt].cpu().numpy())
        return n.value

    # -- LayerKVCache::key_row / value_row / keys / values (proj/src/kv_cache.cpp:57-85)
    def rows(self, seq: int, t0: int = 0, n: int | None = None, raw: bool = False):
        """(K, V) fp32 [n, C] of tokens [t0, t0+n) of sequence seq: the stored
        fused-frame rows (what the reference's key_row/value_row return) or,
        with raw=True, back in the model's frame."""
        torch = self.torch
        if n is None:
            n = int(self.lengths[seq]) - t0 if 0 <= seq < self.cfg.batch else 0
        if not 0 <= seq < self.cfg.batch or t0 < 0 or n < 0 or t0 + n > self.lengths[seq]:
            raise IndexError("cache: token index out of range")
        k = torch.empty(max(n, 1), self.cfg.channels, dtype=torch.float32, device=self.device)
        v = torch.empty_like(k)
        _check(lib().rkv_cache_read(C.byref(self._desc), C.byref(self._view), _ptr(self.perm), seq, t0, n,
                                    1 if raw else 0, _ptr(k), _ptr(v), self._stream()))
        return k[:n], v[:n]

    def key_row(self, seq: int, token: int):
        return self.rows(seq, token, 1)[0][0]

    def value_row(self, seq: int, token: int):
        return self.rows(seq, token, 1)[1][0]

    # -- LayerKVCache::promote_to_sink / route_sinks (proj/src/kv_cache.cpp:43-55, proj/src/sink.cpp:47-63)
    def promote_sinks(self, tokens, k_rows, v_rows):
        """route_sinks for every sequence: tokens = per-sequence lists of token
        indices (or a [B, n] int array, -1 = no entry); k_rows/v_rows = [B, n, C]
        fp16 CUDA tensors holding those tokens' raw (pre-rotation, pre-RoPE)
        rows.  Tokens already sinks are skipped (idempotent).  Out-of-range
        tokens raise IndexError like the reference; a full sidecar raises
        IndexError before anything is changed."""
        torch = self.torch
        B, Cc = self.cfg.batch, self.cfg.channels
        if isinstance(tokens, np.ndarray) and tokens.ndim == 2:
            tok = _np(tokens, np.int64)
        else:
            lists = [list(t) for t in tokens]
            if len(lists) != B:
                raise ValueError("route_sinks: one token list per sequence")
            n = max([len(t) for t in lists] + [1])
            tok = np.full((B, n), -1, np.int64)
            for b, t in enumerate(lists):
                tok[b, :len(t)] = t
        n = tok.shape[1]
        if tok.shape[0] != B:
            raise ValueError("route_sinks: one token list per sequence")
        if k_rows.dtype != torch.float16 or v_rows.dtype != torch.float16 or tuple(k_rows.shape) != (B, n, Cc) \
                or tuple(v_rows.shape) != (B, n, Cc):
            raise ValueError("route_sinks: k_rows/v_rows must be matching [tokens, channels]")
        new = []
        for b in range(B):
            fresh = []
            for t in tok[b]:
                if t == -1:
                    continue
                if t < 0 or t >= self.lengths[b]:
                    raise IndexError("route_sinks: token index out of range")
                if int(t) not in self.sink_tokens[b] and int(t) not in fresh:
                    fresh.append(int(t))
            if self.sink_counts[b] + len(fresh) > self.cfg.max_sinks:
                raise IndexError("cache: sink sidecar capacity exceeded")
            new.append(fresh)
        tok_t = torch.from_numpy(tok).to(self.device)
        k_rows, v_rows = k_rows.contiguous(), v_rows.contiguous()
        _check(lib().rkv_promote_sinks(C.byref(self._desc), C.byref(self._view), _ptr(tok_t), n, _ptr(k_rows),
                                       _ptr(v_rows), None, self._stream()))
        for b in range(B):
            self.sink_tokens[b].update(new[b])
            self.sink_counts[b] += len(new[b])
        self._keep_promote = (tok_t, k_rows, v_rows)
        return [len(x) for x in new]

    # -- LayerKVCache::append (proj/src/kv_cache.cpp:8-22), batched
    def append(self, k, v, sink_flags=None, start_pos=None):
        """k, v: [B, n, C] fp16 CUDA tensors (pre-RoPE, unrotated).
        sink_flags: optional [B, n] bool/uint8.  Appends at each sequence's
        current length unless start_pos ([B] ints) is given."""
        torch = self.torch
        B, Cc = self.cfg.batch, self.cfg.channels
        if k.dtype != torch.float16 or v.dtype != torch.float16:
            raise ValueError("cache append: k and v must be fp16")
        if k.dim() != 3 or k.shape[0] != B or k.shape[2] != Cc or v.shape != k.shape:
            raise ValueError("cache append: row length must equal channel count")
        n = k.shape[1]
        start = self.lengths.copy() if start_pos is None else _np(start_pos, np.int64)
        if np.any(start < 0) or np.any(start + n > self.cfg.max_tokens):
            raise IndexError("cache: token index out of range")
        flags_t = None
        if sink_flags is not None:
            f = torch.as_tensor(sink_flags).to(torch.uint8)
            if tuple(f.shape) != (B, n):
                raise ValueError("sink flags must be [batch, new tokens]")
            add = f.cpu().numpy().astype(np.int64).sum(axis=1)
            if np.any(self.sink_counts + add > self.cfg.max_sinks):
                raise IndexError("cache: sink sidecar capacity exceeded")
            self.sink_counts += add
            fh = f.cpu().numpy()
            for b in range(B):
                self.sink_tokens[b].update(int(start[b]) + np.nonzero(fh[b])[0])
            flags_t = f.to(self.device).contiguous()
        k = k.contiguous()
        v = v.contiguous()
        start_t = torch.from_numpy(start).to(self.device)
        _check(lib().rkv_quantize_kv(C.byref(self._desc), _ptr(k), _ptr(v), _ptr(self.perm), _ptr(flags_t),
                                     _ptr(start_t), n, C.byref(self._view), self._stream()))
        self.lengths = np.maximum(self.lengths, start + n)
        self._keep = (k, v, flags_t, start_t)  # keep inputs alive until the stream consumes them

    def append_fused(self, k_rows, v_rows, sink_flags=None, start_pos=None):
        """LayerKVCache::append in the reference's fused frame (proj/src/
        kv_cache.cpp:8-22 after fuse_weights, proj/src/pipeline.cpp:88-99):
        k_rows = P H_G k (rotated + reordered), v_rows = H_128 v, [B, n, C]
        fp32 (what the reference appends) or fp16 CUDA tensors.  Quantization
        only; sinks and positions as append()."""
        torch = self.torch
        B, Cc = self.cfg.batch, self.cfg.channels
        if k_rows.dtype not in (torch.float32, torch.float16) or v_rows.dtype != k_rows.dtype:
            raise ValueError("cache append_fused: rows must be fp32 or fp16 (both the same)")
        if k_rows.dim() != 3 or k_rows.shape[0] != B or k_rows.shape[2] != Cc or v_rows.shape != k_rows.shape:
            raise ValueError("cache append: row length must equal channel count")
        n = k_rows.shape[1]
        start = self.lengths.copy() if start_pos is None else _np(start_pos, np.int64)
        if np.any(start < 0) or np.any(start + n > self.cfg.max_tokens):
            raise IndexError("cache: token index out of range")
        flags_t = None
        if sink_flags is not None:
            f = torch.as_tensor(sink_flags).to(torch.uint8)
            if tuple(f.shape) != (B, n):
                raise ValueError("sink flags must be [batch, new tokens]")
            add = f.cpu().numpy().astype(np.int64).sum(axis=1)
            if np.any(self.sink_counts + add > self.cfg.max_sinks):
                raise IndexError("cache: sink sidecar capacity exceeded")
            self.sink_counts += add
            fh = f.cpu().numpy()
            for b in range(B):
                self.sink_tokens[b].update(int(start[b]) + np.nonzero(fh[b])[0])
            flags_t = f.to(self.device).contiguous()
        k_rows = k_rows.contiguous()
        v_rows = v_rows.contiguous()
        dtype = ROWS_F32 if k_rows.dtype == torch.float32 else ROWS_F16
        start_t = torch.from_numpy(start).to(self.device)
        _check(lib().rkv_quantize_kv_fused(C.byref(self._desc), _ptr(k_rows), _ptr(v_rows), dtype, _ptr(self.perm),
                                           _ptr(flags_t), _ptr(start_t), n, C.byref(self._view), self._stream()))
        self.lengths = np.maximum(self.lengths, start + n)
        self._keep = (k_rows, v_rows, flags_t, start_t)

    def workspace(self, max_seq_len: int):
        need = lib().rkv_decode_workspace_bytes(C.byref(self._desc), max_seq_len)
        if self._ws is None or self._ws.numel() < need:
            self._ws = self.torch.empty(need, dtype=self.torch.uint8, device=self.device)
        return self._ws, need

    # -- the attention half of decode_step (proj/src/pipeline.cpp:211-261)
    def decode(self, q, seq_len=None, out=None, max_seq_len=None):
        """q: [B, Hq, 128] fp16 pre-RoPE at position seq_len-1.  Returns fp32
        [B, Hq, 128] with V's rotation undone."""
        torch = self.torch
        B, Hq = self.cfg.batch, self.cfg.num_q_heads
        if q.dtype != torch.float16 or tuple(q.shape) != (B, Hq, self.cfg.head_dim):
            raise ValueError("decode_step: input must have d_model elements")
        lens = self.lengths if seq_len is None else _np(seq_len, np.int64)
        if np.any(lens < 1) or np.any(lens > self.lengths):
            raise ValueError("decode_step: position must equal current cache length")
        msl = int(lens.max()) if max_seq_len is None else int(max_seq_len)
        if out is None:
            out = torch.empty((B, Hq, self.cfg.head_dim), dtype=torch.float32, device=self.device)
        ws, need = self.workspace(msl)
        self._lens_t = torch.from_numpy(lens).to(self.device)
        q = q.contiguous()
        _check(lib().rkv_decode_attention(C.byref(self._desc), _ptr(q), _ptr(self._lens_t), msl,
                                          C.byref(self._view), _ptr(self.plan), _ptr(self.rope), _ptr(out),
                                          _ptr(ws), need, self._stream()))
        return out

    # -- sequence-parallel decode (fewer sequences than GPUs)
    def decode_partial(self, q, tok_begin, tok_end, seq_len=None):
        """This rank's share of a decode step: attend to cache tokens
        [tok_begin[b], tok_end[b]) only (sinks excluded), q at position
        seq_len-1.  Returns (ml [B, Hq, 2], o [B, Hq, 128]) fp32 partials in the
        rotated V frame, to be all-gathered and folded by merge_partials."""
        torch = self.torch
        B, Hq = self.cfg.batch, self.cfg.num_q_heads
        if q.dtype != torch.float16 or tuple(q.shape) != (B, Hq, self.cfg.head_dim):
            raise ValueError("decode_step: input must have d_model elements")
        lens = self.lengths if seq_len is None else _np(seq_len, np.int64)
        if np.any(lens < 1) or np.any(lens > self.lengths):
            raise ValueError("decode_step: position must equal current cache length")
        tb, te = _np(tok_begin, np.int64), _np(tok_end, np.int64)
        if tb.shape != (B,) or te.shape != (B,) or np.any(tb < 0) or np.any(te < tb):
            raise ValueError("decode_partial: token ranges must be [B] with 0 <= begin <= end")
        live = tb < np.minimum(te, lens)  # empty ranges need no alignment
        if np.any(live & (tb % 64 != 0)) or np.any(live & (te % 64 != 0) & (te < lens)):
            raise ValueError("decode_partial: range bounds must be multiples of 64 (or the sequence end)")
        span = int(max(1, int((np.minimum(te, lens) - tb).max())))
        ml = torch.empty((B, Hq, 2), dtype=torch.float32, device=self.device)
        o = torch.empty((B, Hq, self.cfg.head_dim), dtype=torch.float32, device=self.device)
        ws, need = self.workspace(span)
        dev = [torch.from_numpy(a).to(self.device) for a in (lens, tb, te)]
        _check(lib().rkv_decode_attention_partial(C.byref(self._desc), _ptr(q.contiguous()), _ptr(dev[0]), _ptr(dev[1]),
                                                  _ptr(dev[2]), span, C.byref(self._view), _ptr(self.plan),
                                                  _ptr(self.rope), _ptr(ml), _ptr(o), _ptr(ws), need, self._stream()))
        return ml, o

    def merge_partials(self, q, parts_ml, parts_o, seq_len=None, out=None):
        """Fold gathered partials ([B, R, Hq, 2], [B, R, Hq, 128]) with the sink
        rows and V's inverse rotation: the decode output for q."""
        torch = self.torch
        B, Hq = self.cfg.batch, self.cfg.num_q_heads
        lens = self.lengths if seq_len is None else _np(seq_len, np.int64)
        R = parts_ml.shape[1]
        if tuple(parts_ml.shape) != (B, R, Hq, 2) or tuple(parts_o.shape) != (B, R, Hq, self.cfg.head_dim):
            raise ValueError("merge_partials: partials must be [B, R, Hq, 2] and [B, R, Hq, d]")
        if out is None:
            out = torch.empty((B, Hq, self.cfg.head_dim), dtype=torch.float32, device=self.device)
        lens_t = torch.from_numpy(lens).to(self.device)
        _check(lib().rkv_decode_merge(C.byref(self._desc), _ptr(q.contiguous()), _ptr(lens_t), R,
                                      _ptr(parts_ml.contiguous()), _ptr(parts_o.contiguous()), C.byref(self._view),
                                      _ptr(self.rope), _ptr(out), self._stream()))
        return out

    def decode_device(self, q, seq_len_t, max_seq_len, out, ws, ws_bytes):
        """Allocation-free decode with device-resident lengths (CUDA-graph safe)."""
        _check(lib().rkv_decode_attention(C.byref(self._desc), _ptr(q), _ptr(seq_len_t), int(max_seq_len),
                                          C.byref(self._view), _ptr(self.plan), _ptr(self.rope), _ptr(out),
                                          _ptr(ws), ws_bytes, self._stream()))
        return out

    def append_device(self, k, v, start_t, sink_flags_t=None):
        """Allocation-free append with device-resident start positions (no
        host mirror update).  Positions past max_tokens are never written (the
        kernel skips them; the device cannot raise)."""
        B, Cc = self.cfg.batch, self.cfg.channels
        if k.dim() != 3 or tuple(k.shape[::2]) != (B, Cc) or v.shape != k.shape:
            raise ValueError("cache append: row length must equal channel count")
        if k.shape[1] > self.cfg.max_tokens or tuple(start_t.shape) != (B,):
            raise IndexError("cache: token index out of range")
        _check(lib().rkv_quantize_kv(C.byref(self._desc), _ptr(k), _ptr(v), _ptr(self.perm), _ptr(sink_flags_t),
                                     _ptr(start_t), k.shape[1], C.byref(self._view), self._stream()))

    def append_fused_device(self, k_rows, v_rows, start_t, sink_flags_t=None):
        """append_fused without the host mirror (device-resident start
        positions, no allocation); fp32 or fp16 rows."""
        B, Cc = self.cfg.batch, self.cfg.channels
        if k_rows.dim() != 3 or tuple(k_rows.shape[::2]) != (B, Cc) or v_rows.shape != k_rows.shape:
            raise ValueError("cache append: row length must equal channel count")
        if k_rows.shape[1] > self.cfg.max_tokens or tuple(start_t.shape) != (B,):
            raise IndexError("cache: token index out of range")
        dtype = ROWS_F32 if k_rows.dtype == self.torch.float32 else ROWS_F16
        _check(lib().rkv_quantize_kv_fused(C.byref(self._desc), _ptr(k_rows), _ptr(v_rows), dtype, _ptr(self.perm),
                                           _ptr(sink_flags_t), _ptr(start_t), k_rows.shape[1], C.byref(self._view),
                                           self._stream()))

    def decode_step(self, k_new, v_new, q):
        """decode_step without projections: append the new token (never a sink,
        proj/src/pipeline.cpp:207-209), then attend over the whole cache."""
        self.append(k_new, v_new)
        return self.decode(q)


def calibrate_reorder_device(cfg: LayerConfig, k, stat: int = STAT_MEAN_ABS):
    """calibrate_reorder from raw fp16 pre-RoPE K rows [rows, C] on the device
    (rotation + per-channel double statistic on the GPU, argsort on the host)
    -> (perm, inverse) int32 numpy, bit-identical to calibrate_reorder(rotate_keys(k))."""
    torch = __import__("torch")
    d = cfg.desc()
    k = k.contiguous().reshape(-1, cfg.channels)
    rows = k.shape[0]
    nws = lib().rkv_calibrate_workspace_bytes(C.byref(d), rows)
    ws = torch.empty(max(nws, 1), dtype=torch.uint8, device=k.device)
    perm = np.empty(cfg.channels, np.int32)
    inv = np.empty(cfg.channels, np.int32)
    _check(lib().rkv_calibrate_reorder_device(C.byref(d), _ptr(k), rows, stat, _ptr(ws), nws, perm.ctypes.data,
                                              inv.ctypes.data,
                                              C.c_void_p(torch.cuda.current_stream(k.device).cuda_stream)))
    return perm, inv


def rotate_keys(cfg: LayerConfig, k):
    """Grouped-head FWHT of raw fp16 K rows [rows, C] on the device -> fp32."""
    torch = __import__("torch")
    d = cfg.desc()
    k = k.contiguous()
    out = torch.empty(k.shape, dtype=torch.float32, device=k.device)
    _check(lib().rkv_rotate_keys(C.byref(d), _ptr(k), k.numel() // cfg.channels, _ptr(out),
                                 C.c_void_p(torch.cuda.current_stream(k.device).cuda_stream)))
    return out
