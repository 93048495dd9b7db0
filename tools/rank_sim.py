"""Multi-GPU scaling estimate on one GPU: time the rank shard an N-GPU run
would give each rank (bench.py's own workloads and sharding), for N = 1, 2,
4, 8, one shard after another on this GPU.  Batch sharding has no collective
on the data path, so each rank's time is its shard's time; the N-GPU step
time is the slowest rank's (the largest shard).  Reports per-rank time and
the implied whole-job throughput and scaling efficiency.  The pool gives one
GPU per call, so this stands in for a real N-GPU run.

    python tools/rank_sim.py            # configs 4 and 3 (decode), 5 (quantize)
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_16383_b200 import sharding  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

dev = torch.device("cuda", 0)
bench.max_over_ranks = lambda vals, dev, world: vals  # one process stands in for every rank
out = {}
for cfg in (4, 3):
    w = WL.CONFIGS[cfg]
    base = None
    for world in (1, 2, 4, 8):
        # the slowest rank holds the largest shard: rank 0 (batch_shard front-loads the remainder)
        _, b_local = sharding.batch_shard(w.batch, world, 0)
        per_layer = bench.decode_bytes(w, b_local, w.tokens, 1)
        layers = max(1, -(-2 * bench.L2_BYTES // per_layer))
        wl = bench.DecodeWorkload(cfg, world, 0, dev, layers=layers)
        st = torch.cuda.current_stream(dev)
        for i in range(max(10, int(100 / max(0.05, 0.7 * b_local / w.batch)))):  # ~100 ms at full clock first
            wl.decode(i)
        ms = statistics.median(bench.time_events(wl.decode, 50, st))
        total = w.batch / (ms / 1e3)
        base = base or total
        rec = {"cfg": cfg, "world": world, "seq_per_rank": b_local, "ms": round(ms, 4), "total_tok_s": round(total, 1),
               "efficiency": round(total / (base * world), 3)}
        print(json.dumps(rec), flush=True)
        out.setdefault(f"cfg{cfg}", []).append(rec)
        del wl
        torch.cuda.empty_cache()
base = None
for world in (1, 2, 4, 8):
    r = bench.bench_quantize_cfg5(dev, world, 0)
    rows = r["token_rows_per_gpu"] * world
    total = rows / (r["ms"] / 1e3)
    base = base or total
    rec = {"cfg": 5, "world": world, "seq_per_rank": r["sequences_per_gpu"], "ms": round(r["ms"], 3),
           "total_rows_s": round(total, 1), "efficiency": round(total / (base * world), 3)}
    print(json.dumps(rec), flush=True)
    out.setdefault("cfg5", []).append(rec)
    torch.cuda.empty_cache()
os.makedirs(os.path.join(bench.ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(bench.ROOT, "gpurun_out", "rank_sim.json"), "w") as f:
    json.dump(out, f, indent=1)
