"""Seeded synthetic inputs with the shapes and distributions of BASELINE.json's
configs (there is no public dataset for this path).

K ~ N(0,1) per channel with `outliers` channels per KV head (a different,
seeded set per head) scaled by U(gain_lo, gain_hi); V, q ~ N(0,1); all fp16,
pre-RoPE.  Sink tokens are the ones a hidden state with magnitude-~100
massive activations flags (proj/src/sink.cpp:14-45): token 0, plus the
seeded "delimiter" positions of config 3.  The channel permutation is
calibrated on 256 seeded tokens of the same distribution (rotated, mean |K|).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    batch: int
    num_q_heads: int
    num_kv_heads: int
    tokens: int
    heads_per_group: int
    rope_base: float
    outliers: int
    gain: tuple
    delimiters: int = 0
    layers: int = 1
    head_dim: int = 128
    extra: dict = field(default_factory=dict)

    @property
    def channels(self) -> int:
        return self.num_kv_heads * self.head_dim


CONFIGS = {
    1: Workload("cfg1-llama2-7b-layer-b1-t4096", 1, 32, 32, 4096, 4, 10000.0, 4, (10.0, 30.0)),
    2: Workload("cfg2-llama2-13b-decode-b16-t4096", 16, 40, 40, 4096, 4, 10000.0, 4, (10.0, 30.0)),
    3: Workload("cfg3-llama3-8b-gqa-b64-t8192", 64, 32, 8, 8192, 2, 500000.0, 6, (20.0, 20.0), delimiters=2),
    4: Workload("cfg4-llama2-7b-longctx-b8-t32768", 8, 32, 32, 32768, 4, 10000.0, 4, (10.0, 30.0)),
    5: Workload("cfg5-llama2-13b-prefill-b128-t2048-l40", 128, 40, 40, 2048, 4, 10000.0, 4, (10.0, 30.0), layers=40),
}


def outlier_gains(w: Workload, seed: int, layer: int = 0) -> np.ndarray:
    """[C] float32 per-channel gain: 1 except `outliers` seeded channels per KV head."""
    rng = np.random.default_rng([seed, 7, layer])
    g = np.ones(w.channels, np.float32)
    for h in range(w.num_kv_heads):
        ch = rng.choice(w.head_dim, size=w.outliers, replace=False)
        g[h * w.head_dim + ch] = rng.uniform(w.gain[0], w.gain[1], size=w.outliers).astype(np.float32)
    return g


def sink_positions(w: Workload, seed: int, tokens: int | None = None) -> list:
    """Token 0 plus seeded delimiter positions (config 3)."""
    t = w.tokens if tokens is None else tokens
    rng = np.random.default_rng([seed, 11])
    pos = [0]
    if w.delimiters and t > 2:
        pos += sorted(int(x) for x in rng.choice(np.arange(1, t), size=min(w.delimiters, t - 1), replace=False))
    return pos


def hidden_with_sinks(w: Workload, seed: int, tokens: int, width: int = 512) -> np.ndarray:
    """[1, tokens, width] hidden state with magnitude ~100 spikes at the sink
    positions; detect_massive_activations(rel=50) recovers them."""
    rng = np.random.default_rng([seed, 13])
    h = rng.standard_normal((1, tokens, width)).astype(np.float32)
    for t in sink_positions(w, seed, tokens):
        h[0, t, rng.integers(0, width)] = 100.0
    return h


def make_kv(w: Workload, seed: int, batch: int, tokens: int, device="cuda", layer: int = 0):
    """(k, v) fp16 [batch, tokens, C] on `device`, seeded."""
    import torch

    gen = torch.Generator(device=device).manual_seed(int(seed) * 1000003 + layer)
    gains = torch.from_numpy(outlier_gains(w, seed, layer)).to(device)
    k = (torch.randn(batch, tokens, w.channels, generator=gen, device=device) * gains).to(torch.float16)
    v = torch.randn(batch, tokens, w.channels, generator=gen, device=device).to(torch.float16)
    return k, v


def make_q(w: Workload, seed: int, batch: int, device="cuda", step: int = 0):
    import torch

    gen = torch.Generator(device=device).manual_seed(int(seed) * 7919 + 17 + step)
    return torch.randn(batch, w.num_q_heads, w.head_dim, generator=gen, device=device).to(torch.float16)


def calibration_perm(w: Workload, seed: int, device="cuda", layer: int = 0, rows: int = 256):
    """Permutation from mean |rotated K| over 256 seeded calibration tokens
    (rotation and channel statistics on the device, rkv_calibrate_reorder_device)."""
    from .rotatekv import LayerConfig, STAT_MEAN_ABS, calibrate_reorder_device

    k, _ = make_kv(w, seed + 100, 1, rows, device=device, layer=layer)
    cfg = LayerConfig(batch=1, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                      heads_per_group=w.heads_per_group, max_tokens=rows, rope_base=w.rope_base)
    perm, _ = calibrate_reorder_device(cfg, k.reshape(rows, w.channels), STAT_MEAN_ABS)
    return perm
