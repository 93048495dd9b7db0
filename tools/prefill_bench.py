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

if os.environ.get("RKV_PF_TRACE"):  # library built with RKV_NVCC_EXTRA=-DRKV_PF_TRACE: hand-off timeline of CTA 0
    import ctypes
    buf = (ctypes.c_longlong * (8 * 256))()
    P.rotatekv.lib().rkv_debug_prefill_trace(buf)
    tr = np.array(buf, dtype=np.int64).reshape(8, 256)
    names = ["s_ready", "p_done", "mma_p_seen", "mma_pv_issued", "mma_qk_start", "prod_v_issue", "r1_s_ready",
             "r1_p_done"]
    t0 = tr[0, 0]
    nt = int((tr[0] != 0).sum())
    print("tile " + " ".join(f"{n:>13}" for n in names))
    for j in range(min(nt, 40)):
        print(f"{j:4d} " + " ".join(f"{int(tr[e, j] - t0) if tr[e, j] else -1:13d}" for e in range(8)))
    d = np.diff(tr[0, 4:nt])
    print("steady tile period (cycles): median", int(np.median(d)), "softmax span median", int(np.median(tr[1, 4:nt] - tr[0, 4:nt])))
    cta = (ctypes.c_ulonglong * (4096 * 4))()
    P.rotatekv.lib().rkv_debug_prefill_cta(cta)
    c = np.array(cta, dtype=np.int64).reshape(4096, 4)
    n = int((c[:, 0] != 0).sum())
    c = c[:n]
    t0 = c[:, 0].min()
    print(f"CTAs {n}: kernel span {(c[:, 3].max() - t0) / 1e3:.1f} us; per CTA (us) median: "
          f"setup+q {np.median(c[:, 1] - c[:, 0]) / 1e3:.2f}, tiles {np.median(c[:, 2] - c[:, 1]) / 1e3:.2f}, "
          f"epilogue {np.median(c[:, 3] - c[:, 2]) / 1e3:.2f}; sum of CTA times / 148 = {(c[:, 3] - c[:, 0]).sum() / 148 / 1e3:.1f} us")
    nq = (c[:, 0] != 0).sum()
    for k in (0, 1, 15, 16, 31):  # grid x index = 31 - qb
        row = c[k]
        print(f"  cta x={k}: setup+q {(row[1] - row[0]) / 1e3:.2f} tiles {(row[2] - row[1]) / 1e3:.2f} epi {(row[3] - row[2]) / 1e3:.2f} us")
