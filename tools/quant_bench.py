"""Quantize-append kernel timing (development tool next to bench.py): one
config-5 layer (128 sequences x 2048 tokens, C = 5120, G = 4, sink at token 0)
through the allocation-free rkv_quantize_kv entry, device-resident inputs,
CUDA events around the launches only.

    python tools/quant_bench.py [stages]      # stages: quantize TMA stage buffers (1 or 2)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

if len(sys.argv) > 1 and hasattr(P, "set_debug_option"):
    P.set_debug_option("quant_stages", int(sys.argv[1]))
if len(sys.argv) > 2:
    P.set_debug_option("quant_vsplit", int(sys.argv[2]))
if len(sys.argv) > 3:
    P.set_debug_option("quant_vcfg", int(sys.argv[3]))
B, T = 128, 2048
w = WL.CONFIGS[5]
perm = WL.calibration_perm(w, 49)
cfg = P.LayerConfig(batch=B, num_q_heads=40, num_kv_heads=40, heads_per_group=4, max_tokens=T, max_sinks=2)
lay = P.RotateKVLayer(cfg, perm)
k, v = WL.make_kv(w, 49, B, T)
flags = torch.zeros(B, T, dtype=torch.uint8, device="cuda")
flags[:, 0] = 1
start = torch.zeros(B, dtype=torch.int64, device="cuda")
times = []
for i in range(6):
    lay.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lay.append_device(k, v, start, flags)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
ms = min(times[1:])
rows = B * T
print(f"quantize {B}x{T} (args {sys.argv[1:]}): {ms:.3f} ms "
      f"(all: {' '.join(f'{t:.3f}' for t in times)}), {rows * 23360 / ms / 1e6:.1f} GB/s")
