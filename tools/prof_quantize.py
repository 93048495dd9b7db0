"""Profiling driver: one config-5-shaped quantize-append (B sequences x T
tokens, C = 5120), timed with CUDA events; used under ncu."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
T = int(sys.argv[2]) if len(sys.argv) > 2 else 256
w = WL.CONFIGS[5]
perm = WL.calibration_perm(w, 49)
cfg = P.LayerConfig(batch=B, num_q_heads=40, num_kv_heads=40, heads_per_group=4, max_tokens=T, max_sinks=2)
lay = P.RotateKVLayer(cfg, perm)
k, v = WL.make_kv(w, 49, B, T)
flags = torch.zeros(B, T, dtype=torch.uint8)
flags[:, 0] = 1
for i in range(3):
    lay.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lay.append(k, v, flags)
    e1.record()
    torch.cuda.synchronize()
    rows = B * T
    ms = e0.elapsed_time(e1)
    print(f"quantize {B}x{T}: {ms:.3f} ms, {rows / ms * 1e3:.3e} tokens/s, {rows * 23360 / ms / 1e6:.1f} GB/s")
