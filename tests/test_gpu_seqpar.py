"""Sequence-parallel decode (fewer sequences than GPUs): the
cache tokens of each sequence are split into rank ranges (token_shard), every
"rank" computes its partial with rkv_decode_attention_partial, and
rkv_decode_merge folds the gathered partials with the sink rows.  On one GPU
the ranks run one after another; the merged output must equal the
single-call decode (same arithmetic, different summation order) and the
oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402
from paper_2501_16383_b200.sharding import token_shard  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.parametrize("hq,hkv,g,world", [(8, 8, 4, 2), (8, 8, 4, 5), (32, 8, 2, 3), (4, 4, 1, 2), (40, 40, 4, 8),
                                              (48, 48, 4, 3),
                                              # GQA 4:1 at G = 4: tensor-core (C = 1024) and generic
                                              # tiled kernel (C = 2048); n = 1024 generic
                                              (32, 8, 4, 3), (64, 16, 4, 2), (16, 16, 8, 2),
                                              # GQA 8:1: head passes of the 4-head kernel
                                              (64, 8, 2, 3), (64, 8, 4, 2),
                                              # more than 8 KV heads; a partial head set
                                              (64, 16, 2, 2), (40, 8, 2, 3), (32, 8, 1, 2)])
def test_partials_merge_to_the_full_decode(oracle, hq, hkv, g, world):
    lens = [700, 129, 64, 1]
    B, T = len(lens), max(lens)
    w = WL.Workload("seqpar", B, hq, hkv, T, g, 10000.0, 4, (10.0, 30.0))
    perm = WL.calibration_perm(w, 5)
    cfg = P.LayerConfig(batch=B, num_q_heads=hq, num_kv_heads=hkv, heads_per_group=g, max_tokens=T + 8, max_sinks=4)
    layer = P.RotateKVLayer(cfg, perm)
    k, v = WL.make_kv(w, 5, B, T)
    flags = torch.zeros(B, T, dtype=torch.uint8)
    flags[:, 0] = 1
    flags[0, 300] = 1
    layer.append(k, v, flags)
    q = WL.make_q(w, 5, B)
    full = layer.decode(q, seq_len=lens).cpu().numpy()
    mls, os_ = [], []
    for r in range(world):
        rng = [token_shard(n, world, r) for n in lens]
        ml, o = layer.decode_partial(q, [a for a, _ in rng], [b for _, b in rng], seq_len=lens)
        mls.append(ml)
        os_.append(o)
    merged = layer.merge_partials(q, torch.stack(mls, 1), torch.stack(os_, 1), seq_len=lens).cpu().numpy()
    for b in range(B):
        assert rel(merged[b], full[b]) < 1e-4, (b, rel(merged[b], full[b]))
    # and the oracle for the longest sequence
    a = {n: t.cpu().numpy() for n, t in layer.arrays().items()}
    n = lens[0]
    want = oracle.decode_attention(a["k_codes"][0, :n].view(np.uint32), a["k_meta"][0, :n].view(np.uint32),
                                   a["v_codes"][0, :n].view(np.uint32), a["v_meta"][0, :n].view(np.uint32),
                                   flags[0, :n].numpy(), k[0, :n].cpu().numpy(), v[0, :n].cpu().numpy(),
                                   q[0].cpu().numpy(), hq, hkv, 128, g, perm, 10000.0)
    assert rel(merged[0], want) < 2e-3


def test_partial_argument_checks():
    w = WL.Workload("seqpar", 1, 8, 8, 64, 4, 10000.0, 4, (10.0, 30.0))
    cfg = P.LayerConfig(batch=1, num_q_heads=8, num_kv_heads=8, heads_per_group=4, max_tokens=128, max_sinks=2)
    layer = P.RotateKVLayer(cfg, WL.calibration_perm(w, 6))
    k, v = WL.make_kv(w, 6, 1, 100)
    layer.append(k, v)
    q = WL.make_q(w, 6, 1)
    with pytest.raises(ValueError):
        layer.decode_partial(q, [10], [64])  # begin not on a 64-token boundary
    with pytest.raises(ValueError):
        layer.decode_partial(q, [64], [0])   # empty-negative range
    ml, o = layer.decode_partial(q, [64], [64])  # empty range: neutral partial
    assert float(ml[0, 0, 1]) == 0.0
