"""Prefill-attention timing on one GPU: a BASELINE-shaped
prompt is quantized into the cache, then rkv_prefill_attention runs the causal
attention of all prompt positions over it (key reconstruction + flash
attention + sink/H_128 combine), timed with CUDA events.

    python tools/prefill_bench.py [cfg] [tokens] [batch]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = WL.CONFIGS[cfg_id]
T = int(sys.argv[2]) if len(sys.argv) > 2 else w.tokens
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
perm = WL.calibration_perm(w, 42 + cfg_id)
cfg = P.LayerConfig(batch=B, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                    heads_per_group=w.heads_per_group, max_tokens=T, max_sinks=4, rope_base=w.rope_base)
layer = P.RotateKVLayer(cfg, perm)
flags = torch.zeros(B, T, dtype=torch.uint8)
flags[:, 0] = 1
for t0 in range(0, T, 1024):
    k, v = WL.make_kv(w, 42 + t0, B, min(1024, T - t0))
    layer.append(k, v, flags[:, t0:t0 + k.shape[1]])
q = torch.randn(B, T, w.num_q_heads, 128, device="cuda").to(torch.float16)
out = layer.prefill_attention(q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
iters = 5
e0.record()
for _ in range(iters):
    layer.prefill_attention(q, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
flops = 4.0 * B * w.num_q_heads * 128 * T * (T + 1) / 2  # causal QK^T + PV, 2 flops per MAC
print(json.dumps({"workload": w.name, "batch": B, "prompt_tokens": T, "ms": round(ms, 3),
                  "prompt_tokens_per_s": B * T / (ms / 1e3), "attention_tflops": flops / (ms / 1e3) / 1e12}))
