"""Prefill (causal) attention over the quantized cache (
proj/src/pipeline.cpp:156-191: reconstruct_cache, then causal
reference_attention, proj/src/attention.cpp:20-49) vs the oracle.

Query row p attends to cache tokens 0..p, so its expected output is the
oracle's decode_attention over the first p+1 tokens with that row as the query
(the decode step's semantics, proj/src/pipeline.cpp:197-261).  Tolerance: the
north star's 2e-3 normalised max error and cosine >= 0.9999, per query row."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402


def build(hq, hkv, g, T, sinks, seed, B=2, base=10000.0):
    w = WL.Workload("prefill", B, hq, hkv, T, g, base, 4, (10.0, 30.0))
    perm = WL.calibration_perm(w, seed)
    cfg = P.LayerConfig(batch=B, num_q_heads=hq, num_kv_heads=hkv, heads_per_group=g, max_tokens=T + 5,
                        max_sinks=4, rope_base=base)
    layer = P.RotateKVLayer(cfg, perm)
    k, v = WL.make_kv(w, seed, B, T)
    flags = torch.zeros(B, T, dtype=torch.uint8)
    for t in sinks:
        if t < T:
            flags[:, t] = 1
    layer.append(k, v, flags)
    gen = torch.Generator(device="cuda").manual_seed(seed + 5)
    q = torch.randn(B, T, hq, 128, generator=gen, device="cuda").to(torch.float16)
    return layer, k, v, flags, q, perm


def expected_rows(oracle, layer, k, v, flags, q, perm, b, rows):
    cfg = layer.cfg
    a = {n: t.cpu().numpy() for n, t in layer.arrays().items()}
    kn, vn, qn, fl = k[b].cpu().numpy(), v[b].cpu().numpy(), q[b].cpu().numpy(), flags[b].numpy()
    out = []
    for p in rows:
        n = p + 1
        out.append(oracle.decode_attention(a["k_codes"][b, :n].view(np.uint32), a["k_meta"][b, :n].view(np.uint32),
                                           a["v_codes"][b, :n].view(np.uint32), a["v_meta"][b, :n].view(np.uint32),
                                           fl[:n], kn[:n], vn[:n], qn[p], cfg.num_q_heads, cfg.num_kv_heads, 128,
                                           cfg.heads_per_group, perm, cfg.rope_base))
    return np.stack(out)


def check(got, want):
    err = float(np.abs(got - want).max() / np.abs(want).max())
    cos = float((got * want).sum() / np.linalg.norm(got) / np.linalg.norm(want))
    assert err <= 2e-3 and cos >= 0.9999, (err, cos)
    return err


@pytest.mark.parametrize("hq,hkv,g,T,sinks,seed", [
    (8, 8, 4, 1, (0,), 0),
    (8, 8, 4, 37, (0,), 1),
    (8, 8, 4, 100, (0, 41, 99), 2),
    (40, 40, 4, 70, (0,), 3),
    (32, 8, 2, 90, (0, 3, 64), 4),
    (32, 8, 2, 33, (), 5),
    # GQA 4:1 at the paper's G = 4 (half-group pairs in the key reconstruction)
    (32, 8, 4, 90, (0, 3, 64), 6), (16, 4, 4, 131, (0,), 7),
    # GQA 8:1 (the decode kernel's head passes; prefill attention is per q head)
    (64, 8, 2, 70, (0, 9), 11), (64, 8, 4, 40, (0,), 12),
    # other ratios (partial head sets on the decode side; prefill attention is per q head)
    (16, 8, 2, 50, (0,), 13), (40, 8, 2, 45, (0, 7), 14), (24, 8, 4, 30, (0,), 15),
    # more than 8 KV heads
    (40, 10, 2, 40, (0,), 16), (64, 16, 4, 33, (0, 5), 17),
    # GQA at G = 1
    (32, 8, 1, 60, (0, 3), 18), (40, 8, 1, 30, (0,), 19),
    (8, 8, 1, 70, (0, 9), 6),
    (8, 8, 2, 45, (0,), 7),
    # the widest tensor-core layer: 12 FWHT groups (C = 6144)
    (48, 48, 4, 50, (0, 7), 8),
    (48, 48, 1, 40, (0,), 9),
    # the widest layer the reference allows: C = 8192 (16 FWHT groups, one CTA per SM)
    (64, 64, 4, 40, (0, 17), 10),
])
def test_prefill_matches_oracle(oracle, hq, hkv, g, T, sinks, seed):
    layer, k, v, flags, q, perm = build(hq, hkv, g, T, sinks, seed)
    out = layer.prefill_attention(q, q_start=np.zeros(2, np.int64)).cpu().numpy()
    for b in range(2):
        want = expected_rows(oracle, layer, k, v, flags, q, perm, b, range(T))
        check(out[b], want)


def test_chunked_queries_and_decode_agree(oracle):
    """A chunk of 20 queries at positions 60..79 of an 80-token cache, and the
    last row against the decode kernel's output for the same query."""
    layer, k, v, flags, q, perm = build(8, 8, 4, 80, (0, 10), 7)
    qc = q[:, 60:80].contiguous()
    out = layer.prefill_attention(qc, q_start=np.full(2, 60, np.int64)).cpu().numpy()
    for b in range(2):
        want = expected_rows(oracle, layer, k, v, flags, q, perm, b, range(60, 80))
        check(out[b], want)
    dec = layer.decode(q[:, 79].contiguous()).cpu().numpy()
    check(out[:, 19], dec)


def test_prefill_rejects_bad_arguments():
    layer, k, v, flags, q, perm = build(8, 8, 4, 16, (0,), 9)
    with pytest.raises(IndexError):
        layer.prefill_attention(q, q_start=np.full(2, 5, np.int64))  # rows past the cache
    with pytest.raises(ValueError):
        layer.prefill_attention(q.float())


@pytest.mark.parametrize("hq,hkv,g", [(96, 24, 2), (12, 3, 1), (64, 64, 8), (24, 8, 8)])
def test_prefill_refuses_shapes_outside_the_tensor_core_path(hq, hkv, g):
    """GQA beyond 16 KV heads, an odd KV-head count at G = 1, and G = 8: ValueError, nothing launched."""
    layer, k, v, flags, q, perm = build(hq, hkv, g, 20, (0,), 1)
    with pytest.raises(ValueError, match="tensor-core path"):
        layer.prefill_attention(q, q_start=np.zeros(2, np.int64))


def test_prefill_rejects_more_than_16_sink_rows():
    """The attention CTA stages at most 16 sink rows: larger max_sinks is refused loudly."""
    w = WL.Workload("prefill", 1, 8, 8, 8, 4, 10000.0, 4, (10.0, 30.0))
    cfg = P.LayerConfig(batch=1, num_q_heads=8, num_kv_heads=8, heads_per_group=4, max_tokens=16, max_sinks=17)
    layer = P.RotateKVLayer(cfg, WL.calibration_perm(w, 3))
    k, v = WL.make_kv(w, 3, 1, 8)
    layer.append(k, v, torch.zeros(1, 8, dtype=torch.uint8))
    q = torch.zeros(1, 8, 8, 128, dtype=torch.float16, device="cuda")
    with pytest.raises(ValueError, match="16 sink rows"):
        layer.prefill_attention(q, q_start=np.zeros(1, np.int64))


def test_prefill_sixteen_sinks_and_ragged_blocks(oracle):
    """16 sink rows (the staging maximum), 150 query rows (a partial 128-row
    block), a second sequence with one sink."""
    B, T = 2, 150
    w = WL.Workload("prefill", B, 8, 8, T, 4, 10000.0, 4, (10.0, 30.0))
    perm = WL.calibration_perm(w, 31)
    cfg = P.LayerConfig(batch=B, num_q_heads=8, num_kv_heads=8, heads_per_group=4, max_tokens=T, max_sinks=16)
    layer = P.RotateKVLayer(cfg, perm)
    k, v = WL.make_kv(w, 31, B, T)
    flags = torch.zeros(B, T, dtype=torch.uint8)
    flags[0, 0:144:9] = 1  # 16 sinks
    flags[1, 0] = 1
    layer.append(k, v, flags)
    gen = torch.Generator(device="cuda").manual_seed(33)
    q = torch.randn(B, T, 8, 128, generator=gen, device="cuda").to(torch.float16)
    out = layer.prefill_attention(q, q_start=np.zeros(B, np.int64)).cpu().numpy()
    for b in range(B):
        rows = list(range(0, T, 7)) + [T - 1]
        want = expected_rows(oracle, layer, k, v, flags, q, perm, b, rows)
        check(out[b, rows], want)


@pytest.mark.parametrize("heads,g,T,sinks,seed", [(8, 4, 48, (0, 20), 11), (4, 4, 9, (0,), 12), (16, 4, 64, (0, 1, 63), 13)])
def test_prefill_matches_reference_prefill(oracle, heads, g, T, sinks, seed):
    """Against the UNMODIFIED reference's prefill (identity projections: each
    token's raw row is its key, value and query; e4m3 scales so the cache is
    the reference's bit for bit)."""
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    C = heads * 128
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((T, C)).astype(np.float16)
    perm = rng.permutation(C).astype(np.int32)
    flags = np.zeros(T, np.uint8)
    for t in sinks:
        flags[t] = 1
    cfg = P.LayerConfig(batch=1, num_q_heads=heads, num_kv_heads=heads, heads_per_group=g, max_tokens=T,
                        max_sinks=4, scale_format=P.SCALE_E4M3_CEIL)
    layer = P.RotateKVLayer(cfg, perm)
    xt = torch.from_numpy(x).cuda()[None]
    layer.append(xt, xt, torch.from_numpy(flags)[None])
    out = layer.prefill_attention(xt.reshape(1, T, heads, 128), q_start=np.zeros(1, np.int64)).cpu().numpy()
    want = oracle.ref_prefill(x.astype(np.float32), flags, perm, heads, 128, g, 10000.0)
    check(out[0].reshape(T, C), want)


@pytest.mark.parametrize("cfg_id,B", [(1, 1), (3, 2)])
def test_prefill_full_size_rows_match_decode(oracle, cfg_id, B):
    """BASELINE shapes at full prompt length (config 1: 32 heads x 4096 tokens;
    config 3: GQA 32/8 heads x 8192 tokens): sampled prompt rows must equal the
    independent decode kernel run at seq_len = p + 1 with the same query (a
    size-independent property), and the first rows the oracle."""
    w = WL.CONFIGS[cfg_id]
    T = w.tokens
    perm = WL.calibration_perm(w, 40 + cfg_id)
    cfg = P.LayerConfig(batch=B, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                        heads_per_group=w.heads_per_group, max_tokens=T, max_sinks=4, rope_base=w.rope_base)
    layer = P.RotateKVLayer(cfg, perm)
    flags = torch.zeros(B, T, dtype=torch.uint8)
    flags[:, 0] = 1
    ks, vs = [], []
    for t0 in range(0, T, 2048):
        k, v = WL.make_kv(w, 40 + t0, B, min(2048, T - t0))
        layer.append(k, v, flags[:, t0:t0 + k.shape[1]])
        if t0 == 0:
            ks.append(k)
            vs.append(v)
    gen = torch.Generator(device="cuda").manual_seed(41)
    q = torch.randn(B, T, w.num_q_heads, 128, generator=gen, device="cuda").to(torch.float16)
    out = layer.prefill_attention(q, q_start=np.zeros(B, np.int64)).cpu().numpy()
    rows = [0, 1, 63, 64, 127, 128, 1000, T // 2 - 1, T // 2, T - 65, T - 1]
    for p in rows:
        dec = layer.decode(q[:, p].contiguous(), seq_len=np.full(B, p + 1, np.int64)).cpu().numpy()
        for b in range(B):
            check(out[b, p], dec[b])
    k0, v0 = ks[0], vs[0]
    want = expected_rows(oracle, layer, k0, v0, flags, q, perm, 0, [0, 5, 70, 300])
    check(out[0, [0, 5, 70, 300]], want)


@pytest.mark.parametrize("hq,hkv,g,T,sinks,seed", [(8, 8, 4, 300, (0, 41), 21), (32, 8, 2, 200, (0,), 22),
                                                   (8, 8, 1, 129, (0, 128), 23)])
def test_prefill_two_sm_pairs_match_oracle(oracle, hq, hkv, g, T, sinks, seed):
    """The opt-in 2-SM mode (cta_group::2 MMAs over CTA pairs, 256 query rows,
    each CTA holding half of every K/V tile) against the oracle."""
    import paper_2501_16383_b200 as P

    P.set_debug_option("prefill_pair", 1)
    try:
        _two_sm_case(oracle, hq, hkv, g, T, sinks, seed)
    finally:
        P.set_debug_option("prefill_pair", 0)


def _two_sm_case(oracle, hq, hkv, g, T, sinks, seed):
    layer, k, v, flags, q, perm = build(hq, hkv, g, T, sinks, seed)
    out = layer.prefill_attention(q, q_start=np.zeros(2, np.int64)).cpu().numpy()
    rows = list(range(0, T, 5)) + [T - 1]
    for b in range(2):
        want = expected_rows(oracle, layer, k, v, flags, q, perm, b, rows)
        check(out[b, rows], want)
