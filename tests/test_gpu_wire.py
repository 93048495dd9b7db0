"""Cache wire format: rkv_cache_export / rkv_cache_import vs
the reference's LayerKVCache::serialize / deserialize (proj/src/kv_cache.cpp:
119-173, blocks proj/src/quant.cpp:139-158).

* e4m3 scales: the GPU cache's bytes equal, byte for byte, the reference's
  serialize() of a LayerKVCache it fills from the same raw rows (fused-frame
  rows, sinks in the fp32 sidecar), and the reference reads them back.
* reference bytes imported into a GPU cache reproduce the GPU's own arrays.
* fp16 scales (RKV_WIRE_FP16_SCALE): export -> import is lossless, decode
  output unchanged.
* errors follow the reference: truncated/empty input -> runtime_error,
  shape mismatch -> invalid_argument."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402


def make_layer(hq, hkv, g, T, fmt, seed, B=2, sinks=(0,)):
    w = WL.Workload("wire", B, hq, hkv, T, g, 10000.0, 4, (10.0, 30.0))
    perm = np.random.default_rng(seed).permutation(hkv * 128).astype(np.int32)
    cfg = P.LayerConfig(batch=B, num_q_heads=hq, num_kv_heads=hkv, heads_per_group=g, max_tokens=T + 8,
                        max_sinks=4, scale_format=fmt)
    layer = P.RotateKVLayer(cfg, perm)
    k, v = WL.make_kv(w, seed, B, T)
    flags = torch.zeros(B, T, dtype=torch.uint8)
    for t in sinks:
        flags[:, t] = 1
    layer.append(k, v, flags)
    return layer, k, v, flags, perm


@pytest.mark.parametrize("hq,hkv,g,T,sinks,seed", [(8, 8, 4, 37, (0,), 0), (32, 8, 2, 20, (0, 5, 19), 1),
                                                   (4, 4, 1, 9, (), 2), (40, 40, 4, 16, (0, 1), 3)])
def test_reference_bytes_identical(oracle, hq, hkv, g, T, sinks, seed):
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    layer, k, v, flags, perm = make_layer(hq, hkv, g, T, P.SCALE_E4M3_CEIL, seed, sinks=sinks)
    for b in range(2):
        ours = layer.serialize(b, P.WIRE_REFERENCE)
        ref = oracle.ref_cache_serialize(k[b].float().cpu().numpy(), v[b].float().cpu().numpy(),
                                         flags[b].numpy(), perm, hkv, 128, g)
        assert len(ours) == len(ref)
        assert ours == ref
        assert oracle.ref_cache_reserialize(ours) == ours  # the reference parses our bytes


def test_import_reference_bytes(oracle):
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    layer, k, v, flags, perm = make_layer(8, 8, 4, 33, P.SCALE_E4M3_CEIL, 5, sinks=(0, 7))
    ref = oracle.ref_cache_serialize(k[1].float().cpu().numpy(), v[1].float().cpu().numpy(), flags[1].numpy(),
                                     perm, 8, 128, 4)
    cfg = layer.cfg
    other = P.RotateKVLayer(cfg, perm)
    assert other.deserialize(ref, 0) == 33
    a, b = layer.arrays(), other.arrays()
    for name in ("k_codes", "v_codes", "k_meta", "v_meta"):
        assert torch.equal(a[name][1, :33], b[name][0, :33]), name
    assert torch.equal(a["sink_mask"][1], b["sink_mask"][0])
    n = int(a["sink_count"][1].item())
    assert int(b["sink_count"][0].item()) == n
    assert torch.equal(a["sink_pos"][1, :n], b["sink_pos"][0, :n])
    # fused-frame fp32 sink rows -> inverse reorder + FWHT -> fp16: within the fp32
    # FWHT's rounding (relative to the row's largest element), not bit-exact
    for name in ("sink_k", "sink_v"):
        x, y = a[name][1, :n].float(), b[name][0, :n].float()
        assert float((x - y).abs().max()) <= 1e-5 * float(x.abs().max()) + 1e-7, name


@pytest.mark.parametrize("hq,hkv,g", [(8, 8, 4), (32, 8, 2)])
def test_fp16_roundtrip_and_decode(hq, hkv, g):
    layer, k, v, flags, perm = make_layer(hq, hkv, g, 40, P.SCALE_FP16_CEIL, 9, sinks=(0, 3))
    data = layer.serialize(0)
    assert data[0] == 0x82  # bits | fp16-scale marker
    other = P.RotateKVLayer(layer.cfg, perm)
    other.deserialize(data, 1)
    other.deserialize(layer.serialize(1), 0)
    a, b = layer.arrays(), other.arrays()
    for name in ("k_codes", "v_codes", "k_meta", "v_meta", "sink_mask"):
        assert torch.equal(a[name][0, :40] if name != "sink_mask" else a[name][0],
                           b[name][1, :40] if name != "sink_mask" else b[name][1]), name
    for name in ("sink_k", "sink_v", "sink_pos"):  # raw fp16 sink rows: lossless
        assert torch.equal(a[name][0, :2], b[name][1, :2]), name
    w = WL.Workload("wire", 2, hq, hkv, 40, g, 10000.0, 4, (10.0, 30.0))
    q = WL.make_q(w, 9, 2)
    qs = torch.stack([q[1], q[0]])
    out_a = layer.decode(q)
    out_b = other.decode(qs)
    assert torch.equal(out_a[0], out_b[1]) and torch.equal(out_a[1], out_b[0])


def test_errors():
    layer, k, v, flags, perm = make_layer(8, 8, 4, 12, P.SCALE_FP16_CEIL, 11)
    data = layer.serialize(0)
    with pytest.raises(RuntimeError, match="truncated"):
        layer.deserialize(data[:-3], 1)
    with pytest.raises(RuntimeError, match="empty"):
        layer.deserialize(b"", 1)
    bad = bytearray(data)
    bad[9:17] = (2048).to_bytes(8, "little")  # channels
    with pytest.raises(ValueError, match="channels"):
        layer.deserialize(bytes(bad), 1)
    with pytest.raises(IndexError, match="sequence"):
        layer.serialize(5)
    # fp16 scales that are not e4m3 values cannot be written in the reference's byte format
    with pytest.raises(ValueError, match="e4m3"):
        layer.serialize(0, P.WIRE_REFERENCE)
