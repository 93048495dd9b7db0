"""Config-5 quantize on one GPU, three input forms: raw fp16 rows (rotation
and reorder in the kernel), and fused-frame fp16 / fp32 rows
(rkv_quantize_kv_fused, quantization only).
    python tools/quant_cfg5.py [raw|f16|f32 ...]"""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
bench.max_over_ranks = lambda vals, dev, world: vals
import paper_2501_16383_b200 as P
for kv in filter(None, os.environ.get("RKV_OPT", "").split(",")):  # experiment switches, e.g. quant_row_buffers=2
    P.set_debug_option(kv.split("=")[0], int(kv.split("=")[1]))
dev = torch.device("cuda", 0)
for f in [None if a == "raw" else a for a in sys.argv[1:]] or (None, "f16", "f32"):
    r = bench.bench_quantize_cfg5(dev, 1, 0, fused=f)
    r.pop("cpu_baseline", None)
    print(json.dumps({"fused": f, "ms": round(r["ms"], 2), "frac": round(r["roofline"]["frac"], 3), "GBs": round(r["roofline"]["achieved"])}), flush=True)
