"""Multi-rank host logic on CPU (gloo, world_size 2): batch sharding gives
every sequence to exactly one rank, rank-local decodes (here the CPU oracle
stands in for the GPU kernel) reassemble bit-identically to the single
process result, and no collective touches the data path before the final
gather.  CPU only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_16383_b200.sharding import batch_shard, gather_batch, shard_rows


def test_batch_shard_partition():
    for B in (0, 1, 3, 16, 64, 65):
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                s, c = batch_shard(B, world, r)
                seen += list(range(s, s + c))
            assert seen == list(range(B))
            sizes = [batch_shard(B, world, r)[1] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        batch_shard(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, inputs, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle

    kc, km, vc, vm, sink, kraw, vraw, q, perm = inputs
    B = kc.shape[0]
    local = []
    for b in range(*(lambda s, c: (s, s + c))(*batch_shard(B, world, rank))):
        local.append(oracle.decode_attention(kc[b], km[b], vc[b], vm[b], sink[b], kraw[b], vraw[b], q[b], 8, 8, 128,
                                             4, perm, 10000.0))
    local_t = torch.from_numpy(np.stack(local)) if local else torch.zeros((0, 8, 128))
    full = gather_batch(local_t, B)
    out_q.put((rank, full.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_decode_matches_single_process(oracle):
    rng = np.random.default_rng(3)
    B, T, H = 3, 20, 8
    C = H * 128
    perm = rng.permutation(C).astype(np.int32)
    kraw = rng.standard_normal((B, T, C)).astype(np.float16)
    vraw = rng.standard_normal((B, T, C)).astype(np.float16)
    q = rng.standard_normal((B, H * 128)).astype(np.float16)
    sink = np.zeros((B, T), np.uint8)
    sink[:, 0] = 1
    packs = [oracle.quantize_kv_rows(kraw[b], vraw[b], H, 128, 4, perm) for b in range(B)]
    kc, km, vc, vm = (np.stack([p[i] for p in packs]) for i in range(4))
    want = np.stack([oracle.decode_attention(kc[b], km[b], vc[b], vm[b], sink[b], kraw[b], vraw[b], q[b], 8, 8, 128, 4,
                                             perm, 10000.0) for b in range(B)])
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    inputs = (kc, km, vc, vm, sink, kraw, vraw, q, perm)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, inputs, out_q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(out_q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert np.array_equal(results[r], want)


def test_shard_rows_views():
    x = np.arange(10 * 3).reshape(10, 3)
    parts = [shard_rows(x, 4, r) for r in range(4)]
    assert np.array_equal(np.concatenate(parts), x)


def test_token_shard_partition():
    from paper_2501_16383_b200.sharding import token_shard

    for T in (0, 1, 63, 64, 65, 700, 4097, 32768):
        for world in (1, 2, 3, 8):
            ranges = [token_shard(T, world, r) for r in range(world)]
            covered = []
            for a, b in ranges:
                assert a <= b and (a == b or a % 64 == 0) and (b % 64 == 0 or b == T)
                covered += list(range(a, b))
            assert covered == list(range(T))
    with pytest.raises(ValueError):
        token_shard(10, 2, 2)


def _seqpar_worker(rank, world, port, logits, values, out_q):
    """Rank-local partial over its token range (a numpy stand-in for
    rkv_decode_attention_partial), all-gathered over gloo, folded with the
    host restatement of rkv_decode_merge's partial fold."""
    from paper_2501_16383_b200.sharding import merge_partials_reference, token_shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = token_shard(len(logits), world, rank)
    s, v = logits[a:b], values[a:b]
    if b > a:
        m = s.max()
        w = np.exp2(s - m)
        part = np.concatenate([[m, w.sum()], (w[:, None] * v).sum(0)])
    else:
        part = np.concatenate([[-np.inf, 0.0], np.zeros(values.shape[1])])
    t = torch.from_numpy(part)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    ps = torch.stack(parts).numpy()
    out_q.put((rank, merge_partials_reference(ps[:, :2], ps[:, 2:])))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sequence_parallel_fold_matches_single_process():
    rng = np.random.default_rng(11)
    T, d = 300, 16
    logits = rng.standard_normal(T) * 6
    values = rng.standard_normal((T, d))
    m = logits.max()
    w = np.exp2(logits - m)
    want = (w[:, None] * values).sum(0) / w.sum()
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seqpar_worker, args=(r, 2, port, logits, values, out_q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(out_q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        mm, ll, oo = results[r]
        assert mm == m
        np.testing.assert_allclose(oo / ll, want, rtol=1e-12, atol=1e-12)


def test_bench_spawns_ranks_dry_run():
    """`bench.py --gpus 2` launches the two ranks itself (no torchrun) and rank
    0 prints one JSON line with n_gpus = 2 (gloo rendezvous on 127.0.0.1)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True
    assert d["max_rank_seen"] == 1.0  # the MAX reduction saw rank 1
    assert d["config"]["batch_per_gpu"] == 4
