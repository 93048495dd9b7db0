import sys, statistics, subprocess, json, os
sys.path.insert(0, '/root/repo')
import torch
import bench
dev = torch.device('cuda', 0)
for world, rank in ((8, 3), (4, 1), (2, 1)):
    from paper_2501_16383_b200 import sharding, workload as WL
    w = WL.CONFIGS[4]
    _, bl = sharding.batch_shard(w.batch, world, rank)
    per_layer = bench.decode_bytes(w, bl, w.tokens, 1)
    layers = max(1, -(-2 * bench.L2_BYTES // per_layer))
    wl = bench.DecodeWorkload(4, world, rank, dev, layers=layers)
    st = torch.cuda.current_stream(dev)
    for i in range(3): wl.decode(i)
    ms = statistics.mean(bench.time_events(wl.decode, 20, st))
    print(json.dumps({"world": world, "rank": rank, "B_local": wl.B, "layers": layers, "ms": ms,
                      "per_gpu_tok_s": wl.B / (ms / 1e3), "implied_total_tok_s": w.batch / (ms / 1e3),
                      "finite": bool(torch.isfinite(wl.out).all())}), flush=True)
    del wl
    torch.cuda.empty_cache()
    r = subprocess.run(["/root/repo/paper_2501_16383_b200/_lib/rkv_e2e_cpp", "--batch", str(bl), "--steps", "10"], capture_output=True, text=True)
    print(r.stdout.strip(), r.stderr.strip()[:200], flush=True)
for cfg in (3,):
    print(json.dumps(bench.bench_extra_decode(cfg, dev, 1, 0, 10)["roofline"]), flush=True)
