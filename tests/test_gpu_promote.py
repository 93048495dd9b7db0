"""promote_to_sink / route_sinks on the device (rkv_promote_sinks):
proj/src/kv_cache.cpp:43-55, proj/src/sink.cpp:47-63.

  * after routing, decode equals the unmodified reference's route_sinks +
    decode_step (e4m3 scales, identity projections) and the oracle;
  * idempotent: promoting a sink again (or twice in one list) changes nothing;
  * out-of-range tokens raise IndexError (std::out_of_range), a full sidecar
    raises before anything changes; the raw C ABI skips such tokens on the
    device without corrupting neighbours.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import ctypes as C  # noqa: E402

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import rotatekv as RK  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

from tests.test_gpu_parity import (COS_TOL, REL_TOL, build_layer, cache_host, cosine, oracle_decode,  # noqa: E402
                                   rel_err, small_workload)


def _rows(k, tokens):
    return torch.stack([k[b, list(t)] for b, t in enumerate(tokens)])


def test_promote_matches_reference_route_sinks(ref):
    w = small_workload(8, 8, 4)
    T = 48
    layer, perm = build_layer(w, 1, T + 1, seed=41, fmt=P.SCALE_E4M3_CEIL)
    k, v = WL.make_kv(w, 41, 1, T + 1)
    x = k[:, T:T + 1]
    sinks = torch.zeros(1, T, dtype=torch.uint8)
    sinks[0, 0] = 1
    layer.append(k[:, :T], v[:, :T], sinks)
    promote = [7, 30, 0]  # token 0 is already a sink: skipped
    n = layer.promote_sinks([promote], _rows(k, [promote]), _rows(v, [promote]))
    assert n == [2]
    assert layer.sink_tokens[0] == {0, 7, 30}
    a = cache_host(layer)
    assert int(a["sink_count"][0]) == 3
    assert not a["k_codes"][0, 7].any() and not a["v_meta"][0, 30].any()
    out = layer.decode_step(x, x, x.reshape(1, 8, 128)).cpu().numpy().reshape(-1)
    want = ref.ref_decode_step_routed(k[0, :T].float().cpu().numpy(), v[0, :T].float().cpu().numpy(),
                                      sinks[0].numpy(), np.array(promote), perm, x[0, 0].float().cpu().numpy(), 8,
                                      128, 4, 10000.0)
    assert rel_err(out, want) < REL_TOL
    assert cosine(out, want) > COS_TOL


def test_promote_batched_vs_oracle_and_idempotent(oracle):
    w = small_workload(40, 40, 4)
    B, T = 3, 300
    layer, perm = build_layer(w, B, T + 4, seed=42, max_sinks=6)
    k, v = WL.make_kv(w, 42, B, T)
    sinks = torch.zeros(B, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    layer.append(k, v, sinks)
    toks = [[5, 5, 250], [299], [0, 1, 2, 3]]
    assert layer.promote_sinks(toks, _rows(k, [t + [0] * (4 - len(t)) for t in toks]),
                               _rows(v, [t + [0] * (4 - len(t)) for t in toks])) == [2, 1, 3]
    before = cache_host(layer)
    q = WL.make_q(w, 42, B)
    out = layer.decode(q).cpu().numpy()
    for b in range(B):
        want = oracle_decode(oracle, layer, before, b, T, q[b].cpu().numpy(), w, perm, k[b].cpu().numpy(),
                             v[b].cpu().numpy())
        assert rel_err(out[b], want) < REL_TOL
        s = {int(x) for x in before["sink_pos"][b, :int(before["sink_count"][b])]}
        assert s == {0} | set(toks[b])
    # again: nothing changes (the reference returns early for sinks)
    assert layer.promote_sinks(toks, _rows(k, [t + [0] * (4 - len(t)) for t in toks]),
                               _rows(v, [t + [0] * (4 - len(t)) for t in toks])) == [0, 0, 0]
    after = cache_host(layer)
    for name in before:  # bit patterns: unused sidecar slots may hold NaN garbage
        assert np.array_equal(before[name].view(np.uint8), after[name].view(np.uint8)), name


def test_promote_errors_and_device_guards():
    w = small_workload(8, 8, 4)
    layer, perm = build_layer(w, 1, 64, seed=43, max_sinks=2)
    k, v = WL.make_kv(w, 43, 1, 40)
    layer.append(k, v, torch.tensor([[1] + [0] * 39], dtype=torch.uint8))
    with pytest.raises(IndexError):  # past the cache length: std::out_of_range
        layer.promote_sinks([[40]], k[:, :1], v[:, :1])
    with pytest.raises(IndexError):  # sidecar capacity 2, one used
        layer.promote_sinks([[3, 4]], k[:, 3:5], v[:, 3:5])
    assert layer.sink_tokens[0] == {0}
    # raw ABI: out-of-range and overflow entries are skipped on the device
    before = cache_host(layer)
    tok = torch.tensor([[-5, 1000, 9, 10]], dtype=torch.int64, device="cuda")
    rows_k, rows_v = k[:, :4].contiguous(), v[:, :4].contiguous()
    got = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = RK.lib().rkv_promote_sinks(C.byref(layer._desc), C.byref(layer._view), tok.data_ptr(), 4,
                                    rows_k.data_ptr(), rows_v.data_ptr(), got.data_ptr(),
                                    C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0
    torch.cuda.synchronize()
    after = cache_host(layer)
    assert int(got[0]) == 1 and int(after["sink_count"][0]) == 2  # token 9 fits, 10 does not
    assert after["sink_pos"][0, 1] == 9
    assert np.array_equal(after["k_codes"][0, 10], before["k_codes"][0, 10])  # stays quantized
    assert not after["k_codes"][0, 9].any()


# ------------------------------------------------------------ row readback

@pytest.mark.parametrize("hq,hkv,g", [(8, 8, 4), (8, 8, 8), (32, 8, 2)])
def test_cache_rows_match_reference_keys_values(ref, hq, hkv, g):
    """rkv_cache_read (STORED frame) == the reference's LayerKVCache::keys() /
    values() bit for bit (e4m3 scales; sinks = fp32 sidecar rows); the RAW
    frame == inverse reorder + FWHT of those rows (the oracle)."""
    w = small_workload(hq, hkv, g)
    T = 40
    layer, perm = build_layer(w, 2, T, seed=61, fmt=P.SCALE_E4M3_CEIL)
    k, v = WL.make_kv(w, 61, 2, T)
    sinks = torch.zeros(2, T, dtype=torch.uint8)
    sinks[:, 0] = 1
    sinks[1, 17] = 1
    layer.append(k, v, sinks)
    for b in range(2):
        ks, vs = layer.rows(b)
        want_k, want_v = ref.ref_cache_rows(k[b].float().cpu().numpy(), v[b].float().cpu().numpy(),
                                            sinks[b].numpy(), perm, hkv, 128, g)
        assert np.array_equal(ks.cpu().numpy(), want_k)
        assert np.array_equal(vs.cpu().numpy(), want_v)
        kr, vr = layer.rows(b, raw=True)
        exp_k = ref.rotate_rows(ref.apply_reorder(want_k, perm, inverse=True), 128, g, hkv)
        exp_v = ref.rotate_rows(want_v, 128, 1, hkv)
        nonsink = [t for t in range(T) if not sinks[b, t]]
        assert np.array_equal(kr.cpu().numpy()[nonsink], exp_k[nonsink])
        assert np.array_equal(vr.cpu().numpy()[nonsink], exp_v[nonsink])
        for t in range(T):  # sinks come back exact in the raw frame
            if sinks[b, t]:
                assert np.array_equal(kr[t].cpu().numpy(), k[b, t].float().cpu().numpy())
    assert torch.equal(layer.key_row(1, 17), layer.rows(1, 17, 1)[0][0])
    with pytest.raises(IndexError):
        layer.rows(0, 35, 10)
