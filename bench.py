#!/usr/bin/env python3
"""Benchmark: decode attention over the 2-bit rotated KV cache (BASELINE
config 2, LLaMA-2-13B-shaped layer: 16 sequences x 40 heads x 128, 4096
cached tokens, G=4) on N B200s, one process per GPU, batch-sharded with no
collective on the data path (weak scaling: every rank holds 16 sequences).

One step = quantize-append of 1 token for each of the rank's 16 sequences
(rkv_quantize_kv, written at position 4096) + decode attention over the 4097
cached tokens (rkv_decode_attention).  The cache (189.5 MB of packed K/V per
step) is larger than the 126 MB L2, so no L2 flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  --impl reference times the reference's own
CPU decode_step (oracle/_ref, compiled from /root/reference) on the host
cores instead, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attn tokens/s and achieved HBM GB/s vs roofline (2-bit KV), 1/2/4/8 B200"
CFG_ID = 2
SEED = 44  # 42 + config index


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-quantize", action="store_true", help="skip the config-5 quantize measurement")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA-graph replays")
    a = ap.parse_args()
    a.warmup = max(a.warmup, 3)
    return a


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def decode_bytes(w, batch, tokens, sinks_per_seq):
    """Algorithmic HBM bytes of one decode launch: per packed
    token 2*(C/4 + 4*C/128), per sink token 2*C*2, plus q (fp16) and out (fp32)."""
    c = w.channels
    packed = (tokens - sinks_per_seq) * 2 * (c // 4 + 4 * c // 128)
    sink = sinks_per_seq * 2 * c * 2
    return batch * (packed + sink) + batch * w.num_q_heads * w.head_dim * (2 + 4)


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml as N

            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _names(self, mask):
        N = self.N
        table = {
            "gpu_idle": getattr(N, "nvmlClocksEventReasonGpuIdle", 0x1),
            "applications_clocks": getattr(N, "nvmlClocksEventReasonApplicationsClocksSetting", 0x2),
            "sw_power_cap": getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sync_boost": getattr(N, "nvmlClocksEventReasonSyncBoost", 0x10),
            "sw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake": getattr(N, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        return {k for k, v in table.items() if mask & v}

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                try:
                    m = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    m = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= self._names(m)
            except Exception:
                break
            time.sleep(0.001)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def cpu_reference_decode(w, perm, nseq, nthreads, steps, warmup):
    """The reference's own decode_step (oracle/_ref) on host threads; falls back
    to the oracle port when the reference library was not built.  Returns
    (seconds per step list, kind, sample description)."""
    import numpy as np

    import oracle

    if oracle.have_ref():
        R = oracle.ref()
        perm32 = np.ascontiguousarray(perm, dtype=np.int32)
        h = R.ref_bench_create(w.num_kv_heads, w.head_dim, w.heads_per_group, w.tokens, nseq,
                               perm32.ctypes.data, w.rope_base, SEED, nthreads)
        if not h:
            raise RuntimeError("ref_bench_create failed")
        try:
            for _ in range(warmup):
                R.ref_bench_step(h, nthreads)
            times = [R.ref_bench_step(h, nthreads) for _ in range(steps)]
        finally:
            R.ref_bench_destroy(h)
        sample = (f"{nseq} sequences x 1 decode step per step (T={w.tokens}, C={w.channels}, G={w.heads_per_group}) "
                  f"through the reference's decode_step (incl. its identity projections), {nthreads} threads, "
                  f"one sequence per thread")
        return times, "reference", sample
    # oracle port: one sequence per step, single thread
    import numpy as np

    rng = np.random.default_rng(SEED)
    T, c = w.tokens, w.channels
    k = rng.standard_normal((T, c)).astype(np.float16)
    v = rng.standard_normal((T, c)).astype(np.float16)
    kc, km, vc, vm = oracle.quantize_kv_rows(k, v, w.num_kv_heads, w.head_dim, w.heads_per_group, perm)
    q = rng.standard_normal(w.num_q_heads * w.head_dim).astype(np.float16)
    s = np.zeros(T, np.uint8)
    s[0] = 1
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        oracle.decode_attention(kc, km, vc, vm, s, k, v, q, w.num_q_heads, w.num_kv_heads, w.head_dim,
                                w.heads_per_group, perm, w.rope_base)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    return times, "port", f"1 sequence x 1 decode step per step (T={T}, C={c}), oracle port, 1 thread"


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    from paper_2501_16383_b200 import workload as WL

    w = WL.CONFIGS[CFG_ID]
    import numpy as np

    perm = np.random.default_rng(SEED).permutation(w.channels).astype(np.int32)
    nthreads = os.cpu_count() or 1
    nseq = min(w.batch, nthreads)
    times, kind, sample = cpu_reference_decode(w, perm, nseq, nthreads, args.steps, args.warmup)
    total = sum(times)
    value = nseq * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(w, world),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": nthreads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(w, world):
    return {
        "workload": w.name,
        "batch_per_gpu": w.batch,
        "global_batch": w.batch * world,
        "cached_tokens": w.tokens,
        "q_heads": w.num_q_heads,
        "kv_heads": w.num_kv_heads,
        "head_dim": w.head_dim,
        "heads_per_group": w.heads_per_group,
        "bits": 2,
        "quant_group": 128,
        "scale": "fp16 ceil",
        "sinks": "token 0 (massive-activation detection)",
        "step": "quantize-append 1 token x batch + decode attention over tokens+1",
        "l2": "no flush: per-step cache bytes (189.5 MB) exceed the 126 MB L2",
        "parallelism": f"batch-sharded x{world}, no collective on the data path",
    }


def bench_quantize_cfg5(dev, world, rank):
    """BASELINE config 5: bulk prefill quantization of a 40-layer
    LLaMA-2-13B-shaped KV cache (128 sequences x 2048 tokens, 40 heads x 128,
    per-layer seeded outlier channels and reorder permutations, sink at token
    0), batch-sharded.  Inputs are generated per layer on the device (214.7 GB
    of fp16 K/V does not fit one GPU); only the quantize-append kernels are
    timed (CUDA events on the stream, positions and sink flags device-resident
    through the allocation-free rkv_quantize_kv entry)."""
    import numpy as np
    import torch

    import paper_2501_16383_b200 as P
    from paper_2501_16383_b200 import sharding
    from paper_2501_16383_b200 import workload as WL

    w = WL.CONFIGS[5]
    _, B = sharding.batch_shard(w.batch, world, rank)
    T, Cc = w.tokens, w.channels
    stream = torch.cuda.current_stream(dev)
    k = torch.empty(B, T, Cc, dtype=torch.float16, device=dev)
    v = torch.empty_like(k)
    flags = torch.zeros(B, T, dtype=torch.uint8, device=dev)
    flags[:, 0] = 1
    start = torch.zeros(B, dtype=torch.int64, device=dev)
    total_ms = 0.0
    layers = []
    for layer in range(w.layers):
        perm = WL.calibration_perm(w, SEED + 5, device=dev, layer=layer)
        cfg = P.LayerConfig(batch=B, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                            heads_per_group=w.heads_per_group, max_tokens=T, max_sinks=2, rope_base=w.rope_base)
        lay = P.RotateKVLayer(cfg, perm, device=dev)
        for b0 in range(0, B, 16):  # seeded per-layer inputs, generated in slices
            kk, vv = WL.make_kv(w, SEED + 5 + 1000 * b0, min(16, B - b0), T, device=dev, layer=layer)
            k[b0:b0 + kk.shape[0]].copy_(kk)
            v[b0:b0 + vv.shape[0]].copy_(vv)
            del kk, vv
        if layer == 0:  # warm-up launch (same shapes)
            lay.append_device(k, v, start, flags)
            lay.reset()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lay.append_device(k, v, start, flags)  # device-resident positions / flags: kernels only
        e1.record(stream)
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        layers.append(lay)  # keep the 40-layer cache resident (755 MB / layer at B=128)
    rows = B * T * w.layers
    bytes_ = rows * (2 * Cc * 2 + 2 * (Cc // 4 + Cc // 32))
    cpu = None
    try:  # the reference's quantize chain (rotate_rows -> apply_reorder -> quantize_token) on the host
        import oracle

        if rank == 0 and oracle.have_ref():
            ns = 256
            kk, vv = WL.make_kv(w, SEED + 5, 1, ns, device=dev)
            kf, vf = kk[0].float().cpu().numpy(), vv[0].float().cpu().numpy()
            t0 = time.perf_counter()
            oracle.ref_quantize_kv_rows(kf, vf, w.num_kv_heads, 128, w.heads_per_group, perm)
            cpu_s = time.perf_counter() - t0
            cpu = {"value": ns / cpu_s, "unit": "token rows/s (K+V)", "cores": 1, "kind": "reference",
                   "sample": f"{ns} token rows of one layer (C={Cc}, G={w.heads_per_group}) through the reference's "
                             "rotate_rows -> apply_reorder -> quantize_token, 1 thread"}
    except Exception as exc:
        cpu = {"error": str(exc)}
    return {"workload": w.name, "sequences_per_gpu": B, "layers": w.layers, "tokens": rows,
            "ms": total_ms, "tokens_per_s_per_gpu": rows / (total_ms / 1e3),
            "hbm_gbs": bytes_ / (total_ms / 1e3) / 1e9, "bytes": bytes_, "cpu_baseline": cpu}


def bench_prefill_cfg1(dev):
    """the attention half of prefill over the quantized cache,
    BASELINE config 1's layer shape (32 heads x 128, G = 4, theta 10000) with a
    4096-token prompt: all 4096 query positions attend causally over the 2-bit
    cache (key reconstruction + flash attention + sink combine), CUDA events.
    Roofline: tensor bound, standard causal-attention flop count (QK^T + PV)
    against the measured dense bf16 peak (the kernel issues 2x that for the
    hi/lo split of Q.K^T)."""
    import torch

    import paper_2501_16383_b200 as P
    from paper_2501_16383_b200 import workload as WL

    w, T, B = WL.CONFIGS[1], 4096, 1
    perm = WL.calibration_perm(w, SEED - 1, device=dev)
    cfg = P.LayerConfig(batch=B, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                        heads_per_group=w.heads_per_group, max_tokens=T, max_sinks=4, rope_base=w.rope_base)
    layer = P.RotateKVLayer(cfg, perm, device=dev)
    flags = torch.zeros(B, T, dtype=torch.uint8)
    flags[:, 0] = 1
    k, v = WL.make_kv(w, SEED - 1, B, T, device=dev)
    layer.append(k, v, flags)
    gen = torch.Generator(device=dev).manual_seed(SEED)
    q = torch.randn(B, T, w.num_q_heads, 128, generator=gen, device=dev).to(torch.float16)
    out = layer.prefill_attention(q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 10
    e0.record(torch.cuda.current_stream(dev))
    for _ in range(iters):
        layer.prefill_attention(q, out=out)
    e1.record(torch.cuda.current_stream(dev))
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    flops = 4.0 * B * w.num_q_heads * 128 * T * (T + 1) / 2
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["bf16_tflops"])
    except Exception:
        peak = 2250.0
    tf = flops / (ms / 1e3) / 1e12
    res = {"workload": "cfg1-llama2-7b-prefill-b1-t4096 (causal attention over the 2-bit cache)", "ms": ms,
           "prompt_tokens_per_s": B * T / (ms / 1e3),
           "roofline": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak}}
    # the reference's own prefill (identity projections) on the host, bounded sample: a 512-token prompt
    try:
        import numpy as np

        import oracle

        if oracle.have_ref():
            Ts = 512
            rng = np.random.default_rng(SEED)
            x = rng.standard_normal((Ts, w.channels)).astype(np.float16)
            fl = np.zeros(Ts, np.uint8)
            fl[0] = 1
            t0 = time.perf_counter()
            oracle.ref_prefill(x.astype(np.float32), fl, perm, w.num_kv_heads, 128, w.heads_per_group, w.rope_base)
            cpu_s = time.perf_counter() - t0
            cfg_s = P.LayerConfig(batch=1, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                                  heads_per_group=w.heads_per_group, max_tokens=Ts, max_sinks=4, rope_base=w.rope_base)
            lay_s = P.RotateKVLayer(cfg_s, perm, device=dev)
            xt = torch.from_numpy(x).to(dev)[None]
            lay_s.append(xt, xt, torch.from_numpy(fl)[None])
            qs = xt.reshape(1, Ts, w.num_q_heads, 128)
            lay_s.prefill_attention(qs)
            torch.cuda.synchronize()
            e0.record(torch.cuda.current_stream(dev))
            for _ in range(iters):
                lay_s.prefill_attention(qs)
            e1.record(torch.cuda.current_stream(dev))
            torch.cuda.synchronize()
            res["cpu_baseline"] = {"value": Ts / cpu_s, "unit": "prompt tokens/s", "cores": 1, "kind": "reference",
                                   "sample": f"1 x {Ts}-token prompt through the reference's prefill (its quantized "
                                             "cache, reconstruct_cache, causal reference_attention; identity "
                                             "projections), 1 thread",
                                   "gpu_same_sample_tokens_per_s": Ts / (e0.elapsed_time(e1) / iters / 1e3)}
    except Exception as exc:
        res["cpu_baseline"] = {"error": str(exc)}
    return res


def run_ours(args):
    import numpy as np
    import torch

    import paper_2501_16383_b200 as P
    from paper_2501_16383_b200 import workload as WL

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    w = WL.CONFIGS[CFG_ID]
    B, T, Hq, D = w.batch, w.tokens, w.num_q_heads, w.head_dim
    seed = SEED + 1000 * rank
    perm = WL.calibration_perm(w, SEED, device=dev)  # one calibrated plan for every rank
    cfg = P.LayerConfig(batch=B, num_q_heads=Hq, num_kv_heads=w.num_kv_heads, heads_per_group=w.heads_per_group,
                        max_tokens=T + 1, max_sinks=4, rope_base=w.rope_base)
    layer = P.RotateKVLayer(cfg, perm, device=dev)
    sink_flags_row = P.detect_massive_activations(WL.hidden_with_sinks(w, seed, T))
    nsinks = int(sink_flags_row.sum())
    flags_all = torch.from_numpy(np.tile(sink_flags_row, (B, 1)))
    chunk = 512
    for t0 in range(0, T, chunk):
        k, v = WL.make_kv(w, seed + t0, B, chunk, device=dev)
        layer.append(k, v, flags_all[:, t0:t0 + chunk])
        del k, v
    torch.cuda.synchronize()

    # step inputs (device resident): a few distinct token/query sets, cycled
    nsets = 4
    kn, vn = zip(*[WL.make_kv(w, seed + 9000 + i, B, 1, device=dev) for i in range(nsets)])
    qs = [WL.make_q(w, seed, B, device=dev, step=i) for i in range(nsets)]
    start_t = torch.full((B,), T, dtype=torch.int64, device=dev)
    len_t = torch.full((B,), T + 1, dtype=torch.int64, device=dev)
    out = torch.empty(B, Hq, D, dtype=torch.float32, device=dev)
    ws, ws_bytes = layer.workspace(T + 1)
    stream = torch.cuda.current_stream(dev)

    def step(i):
        layer.append_device(kn[i % nsets], vn[i % nsets], start_t)
        layer.decode_device(qs[i % nsets], len_t, T + 1, out, ws, ws_bytes)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    # the step as a CUDA-graph-captured pair: one graph per input set
    graphs = None
    if not args.no_graph:
        try:
            graphs = []
            for j in range(nsets):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    step(j)
                graphs.append(g)
            for j in range(nsets):
                graphs[j].replay()
            torch.cuda.synchronize()
        except Exception as e:  # fall back to eager launches, and say so
            print(f"[bench] CUDA graph capture failed ({e}); timing eager launches", file=sys.stderr)
            graphs = None

    # ---- timed region: device-resident inputs, whole steps
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        start.record(stream)
        for i in range(args.steps):
            if graphs is not None:
                graphs[i % nsets].replay()
            else:
                step(i)
        end.record(stream)
        torch.cuda.synchronize()
    barrier()
    elapsed_ms = start.elapsed_time(end)

    # ---- the decode-attention launch alone (roofline of the dominant kernel)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        layer.append_device(kn[i % nsets], vn[i % nsets], start_t)
        ev[i][0].record(stream)
        layer.decode_device(qs[i % nsets], len_t, T + 1, out, ws, ws_bytes)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    decode_ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([elapsed_ms, decode_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, decode_ms = t.tolist()
    ms_per_step = elapsed_ms / args.steps
    value = world * B * args.steps / (elapsed_ms / 1e3)

    # ---- e2e: the same step through the C ABI with HOST buffers (pinned),
    # H2D of the step's new K/V rows and queries, D2H of the outputs, inside
    # the timed region.  Copies run on a copy stream, double buffered, so step
    # i+1's upload and step i-1's download overlap step i's kernels (the
    # serving pattern; every byte still crosses PCIe inside the timed region).
    hk = [x.cpu().pin_memory() for x in kn]
    hv = [x.cpu().pin_memory() for x in vn]
    hq = [x.cpu().pin_memory() for x in qs]
    hout = [torch.empty(B, Hq, D, dtype=torch.float32).pin_memory() for _ in range(2)]
    dk = [torch.empty_like(kn[0]) for _ in range(2)]
    dv = [torch.empty_like(vn[0]) for _ in range(2)]
    dq = [torch.empty_like(qs[0]) for _ in range(2)]
    douts = [torch.empty_like(out) for _ in range(2)]
    copy_s = torch.cuda.Stream(dev)
    up_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    down_done = [torch.cuda.Event() for _ in range(2)]

    def upload(i):
        j = i % 2
        with torch.cuda.stream(copy_s):
            copy_s.wait_event(comp_done[j])  # step i-2 finished reading buffer j
            dk[j].copy_(hk[i % nsets], non_blocking=True)
            dv[j].copy_(hv[i % nsets], non_blocking=True)
            dq[j].copy_(hq[i % nsets], non_blocking=True)
            up_done[j].record(copy_s)

    def e2e_step(i, nsteps):
        j = i % 2
        if i == 0:
            upload(0)
        if i + 1 < nsteps:
            upload(i + 1)
        stream.wait_event(up_done[j])
        stream.wait_event(down_done[j])  # out buffer j downloaded (step i-2)
        layer.append_device(dk[j], dv[j], start_t)
        layer.decode_device(dq[j], len_t, T + 1, douts[j], ws, ws_bytes)
        comp_done[j].record(stream)
        with torch.cuda.stream(copy_s):
            copy_s.wait_event(comp_done[j])
            hout[j].copy_(douts[j], non_blocking=True)
            down_done[j].record(copy_s)

    for i in range(args.warmup):
        e2e_step(i, args.warmup)
    torch.cuda.synchronize()
    barrier()
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record(stream)
    copy_s.wait_event(s2)
    for i in range(args.steps):
        e2e_step(i, args.steps)
    stream.wait_stream(copy_s)  # the last download is inside the timed region
    e2.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = s2.elapsed_time(e2)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()
    e2e_value = world * B * args.steps / (e2e_ms / 1e3)
    h2d = (kn[0].numel() + vn[0].numel() + qs[0].numel()) * 2
    d2h = douts[0].numel() * 4

    # ---- roofline of the dominant kernel (decode attention)
    peak, peak_kind = peak_hbm()
    dbytes = decode_bytes(w, B, T + 1, nsinks)
    achieved = dbytes / (decode_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "decode_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    prefill1 = None
    if rank == 0 and world == 1 and not args.no_quantize:
        try:
            prefill1 = bench_prefill_cfg1(dev)
        except Exception as exc:  # report, never fail the headline line
            prefill1 = {"error": str(exc)}
    quant5 = None
    if not args.no_quantize:
        del layer, ws
        torch.cuda.empty_cache()
        quant5 = bench_quantize_cfg5(dev, world, rank)
        quant5["hbm_frac"] = quant5["hbm_gbs"] / peak_hbm()[0]
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([quant5["ms"]], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            quant5["ms_max_over_ranks"] = t.item()
            quant5["tokens_per_s"] = quant5["tokens"] * world / (t.item() / 1e3)
        else:
            quant5["tokens_per_s"] = quant5["tokens_per_s_per_gpu"]

    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    if rank != 0:
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            nthreads = os.cpu_count() or 1
            nseq = min(B, nthreads)
            times, kind, sample = cpu_reference_decode(w, perm, nseq, nthreads, steps=1, warmup=0)
            cpu = {"value": nseq * len(times) / sum(times), "unit": "tokens/s", "cores": nthreads if kind == "reference" else 1,
                   "kind": kind, "sample": sample}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "unavailable", "sample": str(e)[:200]}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": config_dict(w, world),
        "decode_ms": decode_ms,
        "decode_hbm_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind, "kernel": "rkv_decode_attention",
                     "bytes_per_launch": dbytes},
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": 3 * args.steps,  # quantize_kv, decode split, decode combine per step
        "cuda_graph": graphs is not None,
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
        "quantize_cfg5": quant5,
        "prefill_cfg1": prefill1,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
