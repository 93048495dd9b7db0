#!/usr/bin/env python3
"""Benchmark: decode attention over the 2-bit rotated KV cache on N B200s.

Headline workload (`value`, every N): BASELINE config 4 -- LLaMA-2-7B-shaped
long-context decode, 8 sequences x 32 heads x 128, 32,768 cached tokens,
G = 4, theta 10000 -- batch-sharded over the N ranks (8/N sequences each, one
process per GPU, no collective on the data path; strong scaling: the global
batch of 8 is fixed).  One step = one rkv_decode_attention over every rank's
sequences.  L2: each rank cycles its steps over enough layer caches that the
bytes touched between two visits of a layer exceed 2x the 126 MB L2 (1 layer
at N <= 2, 2 at N = 4, 4 at N = 8), so no step reads another step's lines.

Extra keys on the same line (each with its own HBM roofline): config 2
(16 x 40 heads x 4096 tokens, quantize-append of one token + decode, N = 1),
config 3 (GQA 4:1, 64 sequences x 8192 tokens, batch-sharded 64/N), config 5
(40-layer bulk quantize, 128/N sequences per rank) and the config-1 prefill.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--dry-run]

`--gpus N` without a torchrun environment spawns the N ranks itself (one
process per GPU, RANK/LOCAL_RANK/WORLD_SIZE set, rendezvous on 127.0.0.1);
under torchrun each rank runs directly.  Rank 0 prints ONE JSON line.
`--impl reference` times the reference's own CPU decode_step (oracle/_ref,
compiled from /root/reference; with its DecodeMemo) on the host cores, on a
bounded sample of the same workload.  `--dry-run` exercises the launcher and
the collectives on CPU (gloo) without touching a GPU.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attn tokens/s and achieved HBM GB/s vs roofline (2-bit KV), 1/2/4/8 B200"
HEADLINE_CFG = 4
L2_BYTES = 126 * 1024 * 1024
ARITH = ("codes dequantised to fp16 (one rounding); inverse FWHT on mma.sync tensor cores, fp16 operands with fp32 "
         "accumulate, the second H_16 factor fed an fp16 hi+lo split of the first's fp32 result; RoPE, q.k, online "
         "softmax and P.V accumulation in fp32; P.V weights p*s as fp16 (MHA: one rounding; GQA: hi+lo); sink rows "
         "exact fp16; V's inverse FWHT in fp32")


def seed_of(cfg_id):
    return 42 + cfg_id


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dry-run", action="store_true", help="launcher + collectives on CPU (gloo), no GPU work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="headline only (skip configs 2, 3, 5 and the prefill)")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA-graph replays")
    a = ap.parse_args(argv)
    a.warmup = max(a.warmup, 3)
    a.steps = max(a.steps, 1)
    return a


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n):
    """One process per GPU (the torchrun layout): rank r drives cuda:r."""
    port = str(_free_port())
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    code = 0
    for p in procs:
        code = p.wait() or code
    return code


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def peak_tensor():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]), "measured"
    except Exception:
        return 1590.0, "fallback"


def decode_bytes(w, batch, tokens, sinks_per_seq):
    """Algorithmic HBM bytes of one decode launch: per packed
    token 2*(C/4 + 4*C/128), per sink token 2*C*2, plus q (fp16) and out (fp32)."""
    c = w.channels
    packed = (tokens - sinks_per_seq) * 2 * (c // 4 + 4 * c // 128)
    sink = sinks_per_seq * 2 * c * 2
    return batch * (packed + sink) + batch * w.num_q_heads * w.head_dim * (2 + 4)


def hbm_roofline(nbytes, ms, kernel):
    peak, kind = peak_hbm()
    ach = nbytes / (ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "peak_kind": kind,
            "kernel": kernel, "bytes_per_launch": nbytes, "ms_per_launch": ms}


def source_hash():
    h = hashlib.sha256()
    for f in ("decode_mma.cu", "decode_attention.cu", "generic.cu", "rkv_common.cuh", "rkv_mma.cuh"):
        p = os.path.join(ROOT, "paper_2501_16383_b200", "csrc", f)
        if os.path.exists(p):
            h.update(open(p, "rb").read())
    return h.hexdigest()[:16]


def traffic_for(key):
    """DRAM bytes per launch from the committed ncu capture, only if it was
    taken from the decode sources being timed (hash recorded by
    tools/capture_traffic.py)."""
    tp = os.path.join(ROOT, "profiles", "decode_traffic.json")
    try:
        d = json.load(open(tp))
        if d.get("source_hash") != source_hash():
            return None, "stale (capture predates the timed sources)"
        e = d.get("workloads", {}).get(key)
        return (e.get("dram_bytes_per_launch"), d.get("capture")) if e else (None, "not captured")
    except Exception:
        return None, "no capture"


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


# ---------------------------------------------------------------- CPU reference

def cpu_reference_decode(w, perm, nseq, nthreads, steps, warmup, seed):
    """The reference's own decode_step (oracle/_ref) with its DecodeMemo on
    host threads, one sequence per thread; falls back to the oracle port when
    the reference library was not built.  Returns (seconds per step list,
    kind, sample description, threads used)."""
    import numpy as np

    import oracle

    if oracle.have_ref():
        R = oracle.ref()
        perm32 = np.ascontiguousarray(perm, dtype=np.int32)
        h = R.ref_bench_create(w.num_kv_heads, w.head_dim, w.heads_per_group, w.tokens, nseq, perm32.ctypes.data,
                               w.rope_base, seed, nthreads)
        if not h:
            raise RuntimeError("ref_bench_create failed")
        try:
            R.ref_bench_set_memo(h, 1)
            for _ in range(warmup):  # the first step fills the memo (reconstructs the cache once)
                R.ref_bench_step(h, nthreads)
            times = [R.ref_bench_step(h, nthreads) for _ in range(steps)]
        finally:
            R.ref_bench_destroy(h)
        sample = (f"{nseq} sequences x 1 decode step per step (T={w.tokens}, C={w.channels}, G={w.heads_per_group}) "
                  f"through the reference's decode_step with its DecodeMemo (reconstructed keys memoised across "
                  f"steps, filled during warm-up), identity projections; {min(nthreads, nseq)} threads, one sequence "
                  f"per thread (the reference is single-threaded)")
        return times, "reference", sample, min(nthreads, nseq)
    rng = np.random.default_rng(seed)
    T, c = min(w.tokens, 2048), w.channels
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
            times.append((time.perf_counter() - t0) * w.tokens / T)
    return times, "port", f"1 sequence x 1 decode step (T={T} scaled to {w.tokens}), oracle port, 1 thread", 1


def config_dict(w, world, layers_cycled=1, extra=None):
    d = {
        "workload": w.name,
        "global_batch": w.batch,
        "batch_per_gpu": -(-w.batch // world),
        "cached_tokens": w.tokens,
        "q_heads": w.num_q_heads,
        "kv_heads": w.num_kv_heads,
        "head_dim": w.head_dim,
        "heads_per_group": w.heads_per_group,
        "rope_base": w.rope_base,
        "bits": 2,
        "quant_group": 128,
        "scale": "fp16 ceil",
        "sinks": "token 0 (massive-activation detection)",
        "step": "rkv_decode_attention over every cached token of the rank's sequences",
        "l2": (f"no flush; each rank cycles {layers_cycled} layer cache(s) so the bytes between two visits of a "
               f"layer exceed 2x the 126 MB L2"),
        "parallelism": f"batch-sharded x{world} (one process per GPU), no collective on the data path",
    }
    if extra:
        d.update(extra)
    return d


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import numpy as np

    from paper_2501_16383_b200 import workload as WL

    w = WL.CONFIGS[HEADLINE_CFG]
    perm = np.random.default_rng(seed_of(HEADLINE_CFG)).permutation(w.channels).astype(np.int32)
    nthreads = os.cpu_count() or 1
    nseq = min(w.batch, nthreads)
    times, kind, sample, used = cpu_reference_decode(w, perm, nseq, nthreads, args.steps, args.warmup,
                                                     seed_of(HEADLINE_CFG))
    total = sum(times)
    value = nseq * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded N(0,1) rows, token 0 a sink)",
        "config": config_dict(w, world, extra={"reference_sample": sample}),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": used, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU workloads

class DecodeWorkload:
    """`layers` independent layer caches of a decode config's rank shard,
    filled through rkv_quantize_kv with seeded inputs."""

    def __init__(self, cfg_id, world, rank, dev, layers=1, extra_tokens=0, g=None):
        import dataclasses

        import numpy as np
        import torch

        import paper_2501_16383_b200 as P
        from paper_2501_16383_b200 import sharding
        from paper_2501_16383_b200 import workload as WL

        self.w = w = WL.CONFIGS[cfg_id]
        if g is not None:  # the config's shape at another rotation size (e.g. cfg3 at the paper's G = 4)
            self.w = w = dataclasses.replace(w, heads_per_group=g, name=f"{w.name}-g{g}")
        self.dev = dev
        start, self.B = sharding.batch_shard(w.batch, world, rank)
        seed = seed_of(cfg_id)
        self.perm = WL.calibration_perm(w, seed, device=dev)  # one calibrated plan for every rank
        cfg = P.LayerConfig(batch=self.B, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                            heads_per_group=w.heads_per_group, max_tokens=w.tokens + extra_tokens, max_sinks=4,
                            rope_base=w.rope_base)
        flags_row = P.detect_massive_activations(WL.hidden_with_sinks(w, seed, w.tokens))
        self.nsinks = int(flags_row.sum())
        flags_all = torch.from_numpy(np.tile(flags_row, (self.B, 1)))
        self.layers = []
        chunk = max(256, min(4096, (1 << 27) // max(1, self.B * w.channels)))
        for li in range(layers):
            lay = P.RotateKVLayer(cfg, self.perm, device=dev)
            for t0 in range(0, w.tokens, chunk):
                n = min(chunk, w.tokens - t0)
                k, v = WL.make_kv(w, seed + 1000 * start + 7919 * li + t0, self.B, n, device=dev)
                lay.append(k, v, flags_all[:, t0:t0 + n])
                del k, v
            self.layers.append(lay)
        torch.cuda.synchronize()
        self.qs = [WL.make_q(w, seed + 1000 * start, self.B, device=dev, step=i) for i in range(4)]
        self.len_t = torch.full((self.B,), w.tokens, dtype=torch.int64, device=dev)
        self.out = torch.empty(self.B, w.num_q_heads, w.head_dim, dtype=torch.float32, device=dev)
        self.ws, self.ws_bytes = self.layers[0].workspace(w.tokens)

    def bytes_per_step(self, tokens=None):
        return decode_bytes(self.w, self.B, self.w.tokens if tokens is None else tokens, self.nsinks)

    def decode(self, i, q=None, out=None):
        lay = self.layers[i % len(self.layers)]
        lay.decode_device(self.qs[i % len(self.qs)] if q is None else q, self.len_t, self.w.tokens,
                          self.out if out is None else out, self.ws, self.ws_bytes)


def time_events(fn, steps, stream):
    """Per-launch CUDA-event times (ms) of fn(i) on `stream`."""
    import torch

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for i in range(steps):
        ev[i][0].record(stream)
        fn(i)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def max_over_ranks(vals, dev, world):
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist

    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def bench_extra_decode(cfg_id, dev, world, rank, steps, g=None):
    """A decode config on its rank shard: per-launch CUDA-event time and the
    HBM roofline of rkv_decode_attention (cache bytes > L2 at these shapes, or
    layers cycled).  g: the config's shape at another rotation size."""
    import dataclasses

    import torch

    from paper_2501_16383_b200 import workload as WL

    w = WL.CONFIGS[cfg_id]
    if g is not None:
        w = dataclasses.replace(w, heads_per_group=g, name=f"{w.name}-g{g}")
    from paper_2501_16383_b200 import sharding

    _, b_local = sharding.batch_shard(w.batch, world, rank)
    per_layer = decode_bytes(w, b_local, w.tokens, 1)
    layers = max(1, -(-2 * L2_BYTES // per_layer))
    wl = DecodeWorkload(cfg_id, world, rank, dev, layers=layers, g=g)
    stream = torch.cuda.current_stream(dev)
    for i in range(3):
        wl.decode(i)
    ms = statistics.mean(time_events(wl.decode, steps, stream))
    ms = max_over_ranks([ms], dev, world)[0]
    res = {"workload": w.name, "sequences_per_gpu": wl.B, "layers_cycled": layers, "ms_per_step": ms,
           "tokens_per_s": w.batch / (ms / 1e3),
           "roofline": hbm_roofline(wl.bytes_per_step(), ms, "rkv_decode_attention (decode + combine)")}
    traffic, src = traffic_for(f"cfg{cfg_id}" + (f"_g{g}" if g is not None else ""))
    res["roofline"]["traffic"] = traffic
    res["roofline"]["traffic_source"] = src
    del wl
    torch.cuda.empty_cache()
    return res


def bench_cfg2_step(dev, steps):
    """Config 2 on one GPU: quantize-append of 1 token per sequence (position
    4096) + decode over the 4097 cached tokens, as one CUDA graph per step."""
    import torch

    from paper_2501_16383_b200 import workload as WL

    w = WL.CONFIGS[2]
    wl = DecodeWorkload(2, 1, 0, dev, layers=1, extra_tokens=1)
    lay = wl.layers[0]
    T = w.tokens
    kn, vn = zip(*[WL.make_kv(w, seed_of(2) + 9000 + i, wl.B, 1, device=dev) for i in range(4)])
    start_t = torch.full((wl.B,), T, dtype=torch.int64, device=dev)
    len_t = torch.full((wl.B,), T + 1, dtype=torch.int64, device=dev)
    ws, ws_bytes = lay.workspace(T + 1)
    stream = torch.cuda.current_stream(dev)

    def step(i):
        lay.append_device(kn[i % 4], vn[i % 4], start_t)
        lay.decode_device(wl.qs[i % 4], len_t, T + 1, wl.out, ws, ws_bytes)

    for i in range(3):
        step(i)
    graphs = []
    for j in range(4):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step(j)
        graphs.append(g)
    step_ms = statistics.mean(time_events(lambda i: graphs[i % 4].replay(), steps, stream))

    def dec(i):
        lay.decode_device(wl.qs[i % 4], len_t, T + 1, wl.out, ws, ws_bytes)

    dec_ms = statistics.mean(time_events(dec, steps, stream))
    res = {"workload": w.name, "sequences_per_gpu": wl.B, "ms_per_step": step_ms,
           "tokens_per_s": wl.B / (step_ms / 1e3), "decode_ms": dec_ms,
           "step": "quantize-append 1 token x 16 + decode over 4097 tokens (CUDA graph)",
           "roofline": hbm_roofline(decode_bytes(w, wl.B, T + 1, wl.nsinks), dec_ms,
                                    "rkv_decode_attention (decode + combine)")}
    traffic, src = traffic_for("cfg2")
    res["roofline"]["traffic"] = traffic
    res["roofline"]["traffic_source"] = src
    del wl, graphs
    torch.cuda.empty_cache()
    return res


def bench_quantize_cfg5(dev, world, rank, fused=None):
    """BASELINE config 5: bulk prefill quantization of a 40-layer
    LLaMA-2-13B-shaped KV cache (128 sequences x 2048 tokens, 40 heads x 128,
    per-layer seeded outlier channels and reorder permutations, sink at token
    0), batch-sharded 128/N.  Inputs are generated per layer on the device
    (214.7 GB of fp16 K/V does not fit one GPU); only the quantize-append
    kernels are timed (CUDA events, device-resident positions and flags).
    fused = "f16" / "f32": the same rows appended in the fused frame
    (rkv_quantize_kv_fused: quantization only), as fp16 or fp32
    rows -- the generated values stand in for K' / V'."""
    import torch

    import paper_2501_16383_b200 as P
    from paper_2501_16383_b200 import sharding
    from paper_2501_16383_b200 import workload as WL

    w = WL.CONFIGS[5]
    seed = seed_of(5)
    _, B = sharding.batch_shard(w.batch, world, rank)
    T, Cc = w.tokens, w.channels
    stream = torch.cuda.current_stream(dev)
    k = torch.empty(B, T, Cc, dtype=torch.float32 if fused == "f32" else torch.float16, device=dev)
    v = torch.empty_like(k)
    append = (lambda lay: lay.append_device(k, v, start, flags)) if fused is None else \
        (lambda lay: lay.append_fused_device(k, v, start, flags))
    flags = torch.zeros(B, T, dtype=torch.uint8, device=dev)
    flags[:, 0] = 1
    start = torch.zeros(B, dtype=torch.int64, device=dev)
    total_ms = 0.0
    layers = []
    for layer in range(w.layers):
        perm = WL.calibration_perm(w, seed, device=dev, layer=layer)
        cfg = P.LayerConfig(batch=B, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                            heads_per_group=w.heads_per_group, max_tokens=T, max_sinks=2, rope_base=w.rope_base)
        lay = P.RotateKVLayer(cfg, perm, device=dev)
        for b0 in range(0, B, 16):  # seeded per-layer inputs, generated in slices
            kk, vv = WL.make_kv(w, seed + 1000 * b0, min(16, B - b0), T, device=dev, layer=layer)
            k[b0:b0 + kk.shape[0]].copy_(kk)
            v[b0:b0 + vv.shape[0]].copy_(vv)
            del kk, vv
        if layer == 0:  # warm-up launch (same shapes)
            append(lay)
            lay.reset()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        append(lay)
        e1.record(stream)
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        layers.append(lay)  # keep the 40-layer cache resident
    total_ms = max_over_ranks([total_ms], dev, world)[0]
    rows = B * T * w.layers
    bytes_ = rows * (2 * Cc * k.element_size() + 2 * (Cc // 4 + Cc // 32))
    res = {"workload": w.name, "sequences_per_gpu": B, "layers": w.layers, "token_rows_per_gpu": rows,
           "ms": total_ms, "tokens_per_s": w.batch * T * w.layers / (total_ms / 1e3),
           "roofline": hbm_roofline(bytes_, total_ms, "rkv_quantize_kv (40 launches)" if fused is None else
                                    f"rkv_quantize_kv_fused, {fused} rows (40 launches)")}
    if fused is not None:
        res["input"] = f"fused-frame rows ({fused}): quantization only, no rotation or reorder"
        del layers, k, v
        torch.cuda.empty_cache()
        return res
    try:  # the reference's quantize chain (rotate_rows -> apply_reorder -> quantize_token) on the host
        import oracle

        if rank == 0 and world == 1 and oracle.have_ref():
            ns = 256
            kk, vv = WL.make_kv(w, seed, 1, ns, device=dev)
            kf, vf = kk[0].float().cpu().numpy(), vv[0].float().cpu().numpy()
            t0 = time.perf_counter()
            oracle.ref_quantize_kv_rows(kf, vf, w.num_kv_heads, 128, w.heads_per_group, perm)
            cpu_s = time.perf_counter() - t0
            res["cpu_baseline"] = {"value": ns / cpu_s, "unit": "token rows/s (K+V, one layer)", "cores": 1,
                                   "kind": "reference",
                                   "sample": f"{ns} token rows of one layer (C={Cc}, G={w.heads_per_group}) through "
                                             "the reference's rotate_rows -> apply_reorder -> quantize_token, 1 thread"}
    except Exception as exc:
        res["cpu_baseline"] = {"error": str(exc)[:200]}
    del layers, k, v
    torch.cuda.empty_cache()
    return res


def bench_prefill_cfg1(dev):
    """the attention half of prefill over the quantized cache,
    BASELINE config 1's layer shape (32 heads x 128, G = 4, theta 10000) with a
    4096-token prompt (key reconstruction + tcgen05 flash attention + sink
    combine), CUDA events.  Roofline: tensor bound, standard causal-attention
    flop count (QK^T + PV) against the measured dense bf16 peak."""
    import numpy as np
    import torch

    import paper_2501_16383_b200 as P
    from paper_2501_16383_b200 import workload as WL

    w, T, B = WL.CONFIGS[1], 4096, 1
    perm = WL.calibration_perm(w, seed_of(1), device=dev)
    cfg = P.LayerConfig(batch=B, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                        heads_per_group=w.heads_per_group, max_tokens=T, max_sinks=4, rope_base=w.rope_base)
    layer = P.RotateKVLayer(cfg, perm, device=dev)
    flags = torch.zeros(B, T, dtype=torch.uint8)
    flags[:, 0] = 1
    k, v = WL.make_kv(w, seed_of(1), B, T, device=dev)
    layer.append(k, v, flags)
    gen = torch.Generator(device=dev).manual_seed(seed_of(1))
    q = torch.randn(B, T, w.num_q_heads, 128, generator=gen, device=dev).to(torch.float16)
    out = layer.prefill_attention(q)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    ms = statistics.mean(time_events(lambda i: layer.prefill_attention(q, out=out), 10, stream))
    flops = 4.0 * B * w.num_q_heads * 128 * T * (T + 1) / 2
    peak, kind = peak_tensor()
    tf = flops / (ms / 1e3) / 1e12
    res = {"workload": "cfg1-llama2-7b-prefill-b1-t4096 (causal attention over the 2-bit cache)", "ms": ms,
           "prompt_tokens_per_s": B * T / (ms / 1e3),
           "roofline": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                        "peak_kind": kind, "kernel": "rkv_prefill_attention (4 launches)",
                        "flops_per_launch": flops}}
    try:
        import oracle

        if oracle.have_ref():
            Ts = 512
            rng = np.random.default_rng(seed_of(1))
            x = rng.standard_normal((Ts, w.channels)).astype(np.float16)
            fl = np.zeros(Ts, np.uint8)
            fl[0] = 1
            t0 = time.perf_counter()
            oracle.ref_prefill(x.astype(np.float32), fl, perm, w.num_kv_heads, 128, w.heads_per_group, w.rope_base)
            cpu_s = time.perf_counter() - t0
            res["cpu_baseline"] = {"value": Ts / cpu_s, "unit": "prompt tokens/s", "cores": 1, "kind": "reference",
                                   "sample": f"1 x {Ts}-token prompt through the reference's prefill (its quantized "
                                             "cache, reconstruct_cache, causal reference_attention; identity "
                                             "projections), 1 thread"}
    except Exception as exc:
        res["cpu_baseline"] = {"error": str(exc)[:200]}
    return res


def run_dry(args):
    """The multi-rank harness without a GPU: rendezvous (gloo), barrier and the
    max-over-ranks reduction, then rank 0's line."""
    rank, _, world = dist_env()
    elapsed = 0.0
    if world > 1:
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo")
        dist.barrier()
        t = torch.tensor([float(rank)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = t.item()
        dist.destroy_process_group()
    if rank == 0:
        from paper_2501_16383_b200 import workload as WL

        w = WL.CONFIGS[HEADLINE_CFG]
        print(json.dumps({"metric": METRIC, "value": None, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "dry_run": True, "max_rank_seen": elapsed,
                          "config": config_dict(w, world)}), flush=True)


def run_ours(args):
    import torch

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    from paper_2501_16383_b200 import sharding
    from paper_2501_16383_b200 import workload as WL

    w = WL.CONFIGS[HEADLINE_CFG]
    _, b_local = sharding.batch_shard(w.batch, world, rank)
    per_layer = decode_bytes(w, b_local, w.tokens, 1)
    layers = max(1, -(-2 * L2_BYTES // per_layer))  # bytes between two visits of a layer >= 2 x L2
    layers = max(max_over_ranks([float(layers)], dev, world)[0], 1)
    layers = int(layers)
    wl = DecodeWorkload(HEADLINE_CFG, world, rank, dev, layers=layers)
    stream = torch.cuda.current_stream(dev)
    for i in range(args.warmup):
        wl.decode(i)
    torch.cuda.synchronize()

    graphs = None
    if not args.no_graph:  # one graph per (layer, query set): decode + combine
        try:
            graphs = {}
            for i in range(len(wl.layers) * len(wl.qs)):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    wl.decode(i)
                graphs[i] = g
            for g in graphs.values():
                g.replay()
            torch.cuda.synchronize()
        except Exception as e:
            print(f"[bench] CUDA graph capture failed ({e}); timing eager launches", file=sys.stderr)
            graphs = None
    ncyc = len(wl.layers) * len(wl.qs)

    def step(i):
        if graphs is not None:
            graphs[i % ncyc].replay()
        else:
            wl.decode(i)

    # ---- timed region: device-resident inputs, K whole steps back to back
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        start.record(stream)
        for i in range(args.steps):
            step(i)
        end.record(stream)
        torch.cuda.synchronize()
    barrier()
    elapsed_ms = start.elapsed_time(end)
    # ---- the rkv_decode_attention launch alone (roofline of the dominant kernel)
    launch_ms = time_events(step, args.steps, stream)
    decode_ms = statistics.mean(launch_ms)
    elapsed_ms, decode_ms = max_over_ranks([elapsed_ms, decode_ms], dev, world)
    ms_per_step = elapsed_ms / args.steps
    value = w.batch * args.steps / (elapsed_ms / 1e3)

    # ---- e2e: the same step through the public API (C ABI via the Python host
    # layer) with HOST buffers: per step the H2D of the rank's queries from
    # pinned memory and the D2H of its outputs are inside the timed region;
    # copies on a copy stream, double buffered, so step i+1's upload and step
    # i-1's download overlap step i's kernels (the serving pattern).
    hq = [x.cpu().pin_memory() for x in wl.qs]
    hout = [torch.empty_like(wl.out, device="cpu").pin_memory() for _ in range(2)]
    dq = [torch.empty_like(wl.qs[0]) for _ in range(2)]
    douts = [torch.empty_like(wl.out) for _ in range(2)]
    copy_s = torch.cuda.Stream(dev)
    up_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    down_done = [torch.cuda.Event() for _ in range(2)]

    def upload(i):
        j = i % 2
        with torch.cuda.stream(copy_s):
            copy_s.wait_event(comp_done[j])  # step i-2 finished reading buffer j
            dq[j].copy_(hq[i % len(hq)], non_blocking=True)
            up_done[j].record(copy_s)

    def e2e_step(i, nsteps):
        j = i % 2
        if i == 0:
            upload(0)
        if i + 1 < nsteps:
            upload(i + 1)
        stream.wait_event(up_done[j])
        stream.wait_event(down_done[j])  # out buffer j downloaded (step i-2)
        wl.decode(i, q=dq[j], out=douts[j])
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
    e2e_ms = max_over_ranks([s2.elapsed_time(e2)], dev, world)[0]
    e2e_value = w.batch * args.steps / (e2e_ms / 1e3)
    h2d = wl.qs[0].numel() * 2 * world
    d2h = wl.out.numel() * 4 * world

    # ---- e2e_cpp: the same step through the C++ API (rotatekv.hpp DeviceLayerCache)
    e2e_cpp = None
    try:
        from paper_2501_16383_b200 import build as BLD

        exe = BLD.E2E_CPP
        if os.path.exists(exe):
            r = subprocess.run([exe, "--batch", str(wl.B), "--q-heads", str(w.num_q_heads), "--kv-heads",
                                str(w.num_kv_heads), "--group", str(w.heads_per_group), "--tokens", str(w.tokens),
                                "--steps", str(args.steps), "--warmup", str(args.warmup), "--device", str(local),
                                "--seed", str(seed_of(HEADLINE_CFG))], capture_output=True, text=True, timeout=600)
            d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
            ms_cpp = max_over_ranks([d["ms"]], dev, world)[0]
            e2e_cpp = {"value": w.batch * args.steps / (ms_cpp / 1e3), "unit": "tokens/s",
                       "h2d_bytes_per_step": d["h2d_bytes_per_step"] * world,
                       "d2h_bytes_per_step": d["d2h_bytes_per_step"] * world, "finite": d["finite"],
                       "path": "C++ API (rotatekv.hpp DeviceLayerCache::decode_attention), pinned host q in / "
                               "fp32 out per step on a copy stream, double buffered (as e2e), one process per GPU "
                               "(paper_2501_16383_b200/csrc/e2e_cpp.cu)"}
        else:
            max_over_ranks([0.0], dev, world)
    except Exception as exc:
        e2e_cpp = {"error": str(exc)[:200]}
    roof = hbm_roofline(wl.bytes_per_step(), decode_ms, "rkv_decode_attention (decode_mma_kernel + combine), per rank")
    roof["traffic"], roof["traffic_source"] = traffic_for(f"cfg{HEADLINE_CFG}")
    del wl, graphs
    torch.cuda.empty_cache()

    extras = {}
    if not args.no_extras:
        for key, fn in (("cfg3", lambda: bench_extra_decode(3, dev, world, rank, min(args.steps, 30))),
                        # GQA 4:1 at the paper's default rotation G = 4 (tensor-core half-group pairs)
                        ("cfg3_g4", lambda: bench_extra_decode(3, dev, world, rank, min(args.steps, 10), g=4)),
                        ("cfg2", (lambda: bench_cfg2_step(dev, min(args.steps, 30))) if world == 1 else None),
                        ("prefill_cfg1", (lambda: bench_prefill_cfg1(dev)) if world == 1 and rank == 0 else None),
                        ("quantize_cfg5", lambda: bench_quantize_cfg5(dev, world, rank)),
                        # the same rows in the reference's fused frame (quantization only): fp32 rows
                        # (what LayerKVCache::append receives) and fp16 rows
                        ("quantize_cfg5_fused", lambda: bench_quantize_cfg5(dev, world, rank, fused="f32")),
                        ("quantize_cfg5_fused_f16", lambda: bench_quantize_cfg5(dev, world, rank, fused="f16"))):
            if fn is None:
                continue
            try:
                extras[key] = fn()
            except Exception as exc:  # report, never fail the headline line
                extras[key] = {"error": str(exc)[:300]}
                torch.cuda.empty_cache()

    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    if rank != 0:
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            import numpy as np

            perm = np.random.default_rng(seed_of(HEADLINE_CFG)).permutation(w.channels).astype(np.int32)
            nthreads = os.cpu_count() or 1
            nseq = min(w.batch, nthreads)
            times, kind, sample, used = cpu_reference_decode(w, perm, nseq, nthreads, steps=2, warmup=1,
                                                             seed=seed_of(HEADLINE_CFG))
            cpu = {"value": nseq * len(times) / sum(times), "unit": "tokens/s", "cores": used, "kind": kind,
                   "sample": sample}
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
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "arith": ARITH,
        "data": "synthetic (seeded; BASELINE distributions: outlier channels x10-30, token-0 sink)",
        "config": config_dict(w, world, layers),
        "decode_ms": decode_ms,
        "decode_hbm_gbs_per_gpu": roof["achieved"],
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "Python host layer -> C ABI rkv_decode_attention, pinned host q in / fp32 out per step"},
        "e2e_cpp": e2e_cpp,
        "gpu_launches": 2 * args.steps,  # decode_mma_kernel + decode_combine_kernel per step
        "cuda_graph": not args.no_graph,
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
        "source_hash": source_hash(),
    }
    line.update(extras)
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, _, world = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
