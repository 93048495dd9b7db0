"""Decode-kernel timing over the BASELINE decode configs on one GPU (a
development tool next to bench.py): fills a seeded 2-bit cache per config and
times rkv_decode_attention alone with CUDA events.

    python tools/decode_sweep.py [cfg ...]      (default: 2 3 4; "2g1" = config 2 with G = 1)
    RKV_DECODE_KERNEL=simt python tools/decode_sweep.py   # the CUDA-core kernel (debug option)

cfg 4 (8 x 32768 tokens) is timed at full size; cfg 3 at batch 64 x 8192.
"""
import dataclasses
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402


def decode_bytes(w, B, T, nsinks):
    c = w.channels
    return B * ((T - nsinks) * 2 * (c // 4 + 4 * c // 128) + nsinks * 4 * c) + B * w.num_q_heads * 128 * 6


def run(cfg_id, iters=20, g=None, warm=3, h=None, b=None, qh=None, kv=None):
    w = WL.CONFIGS[cfg_id]
    if kv is not None:  # KV heads only (e.g. 16: GQA past 8 KV heads)
        w = dataclasses.replace(w, num_kv_heads=kv, name=f"{w.name}-k{kv}")
    if qh is not None:  # q heads only (another GQA ratio, e.g. 64 over 8 KV heads)
        w = dataclasses.replace(w, num_q_heads=qh, name=f"{w.name}-q{qh}")
    if b is not None:  # a rank shard's batch (e.g. config 4 at 8 GPUs: b = 1)
        w = dataclasses.replace(w, batch=b, name=f"{w.name}-b{b}")
    if g is not None:  # same shape with another rotation group size (e.g. the reference default G = 1)
        w = dataclasses.replace(w, heads_per_group=g, name=f"{w.name}-g{g}")
    if h is not None:  # same shape with h q heads and h KV heads (e.g. 64: C = 8192)
        w = dataclasses.replace(w, num_q_heads=h, num_kv_heads=h, name=f"{w.name}-h{h}")
    dev = torch.device("cuda", 0)
    B, T = w.batch, w.tokens
    perm = WL.calibration_perm(w, 42 + cfg_id, device=dev)
    cfg = P.LayerConfig(batch=B, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                        heads_per_group=w.heads_per_group, max_tokens=T, max_sinks=4, rope_base=w.rope_base)
    layer = P.RotateKVLayer(cfg, perm, device=dev)
    flags_row = np.zeros(T, np.uint8)
    for t in WL.sink_positions(w, 42 + cfg_id, T):
        flags_row[t] = 1
    flags = torch.from_numpy(np.tile(flags_row, (B, 1)))
    chunk = max(1, min(T, (1 << 26) // (B * w.channels)))
    for t0 in range(0, T, chunk):
        k, v = WL.make_kv(w, 42 + cfg_id + t0, B, min(chunk, T - t0), device=dev)
        layer.append(k, v, flags[:, t0:t0 + k.shape[1]])
        del k, v
    q = WL.make_q(w, 42 + cfg_id, B, device=dev)
    lens = torch.full((B,), T, dtype=torch.int64, device=dev)
    out = torch.empty(B, w.num_q_heads, 128, dtype=torch.float32, device=dev)
    ws, wsb = layer.workspace(T)
    for _ in range(warm):
        layer.decode_device(q, lens, T, out, ws, wsb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        layer.decode_device(q, lens, T, out, ws, wsb)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    nb = decode_bytes(w, B, T, int(flags_row.sum()))
    return {"cfg": cfg_id, "workload": w.name, "kernel": os.environ.get("RKV_DECODE_KERNEL", "default"),
            "us": round(us, 1), "GB/s": round(nb / us / 1e3, 1), "bytes": nb}


if __name__ == "__main__":
    if os.environ.get("RKV_DECODE_KERNEL") == "simt":
        P.set_debug_option("decode_kernel_simt", 1)
    for kv in filter(None, os.environ.get("RKV_OPT", "").split(",")):  # e.g. RKV_OPT=mha_pipe=1
        k_, v_ = kv.split("=")
        P.set_debug_option(k_, int(v_))
    # "2" = config 2; "2g1" = config 2's shape with G = 1; "2h64" = with 64 (q = KV) heads;
    # "4b1" = config 4 with batch 1; "3q64" = config 3 with 64 q heads (GQA 8:1);
    # "3k16q64" = config 3 with 16 KV and 64 q heads
    # --profile: one warm-up and one timed launch per config (for ncu captures)
    prof = "--profile" in sys.argv
    ids = [a for a in sys.argv[1:] if not a.startswith("--")] or ["2", "3", "4"]
    for a in ids:
        a, _, qs = a.partition("q")
        a, _, ks = a.partition("k")
        a, _, bs = a.partition("b")
        a, _, h = a.partition("h")
        cfg, _, g = a.partition("g")
        print(json.dumps(run(int(cfg), g=int(g) if g else None, iters=1 if prof else 20, warm=1 if prof else 3,
                             h=int(h) if h else None, b=int(bs) if bs else None, qh=int(qs) if qs else None,
                             kv=int(ks) if ks else None)),
              flush=True)
