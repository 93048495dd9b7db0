"""Device-side guards (the device cannot throw):
  * rkv_quantize_kv never writes rows at positions >= max_tokens, and a full
    sink sidecar keeps the token quantized (mask clear, count unchanged);
  * a decode with a layer plan built for another shape or kernel kind
    returns NaN instead of silently wrong attention;
  * rkv_rotate_keys takes calibration sets above 65,535 rows.
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import rotatekv as RK  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

from tests.test_gpu_parity import build_layer, cache_host, small_workload  # noqa: E402


def test_append_device_skips_rows_past_capacity(oracle):
    w = small_workload(8, 8, 4)
    B, T = 2, 32
    layer, perm = build_layer(w, B, T, seed=51, max_sinks=1)
    k, v = WL.make_kv(w, 51, B, 8)
    # sequence 0 writes at 28..35 (4 rows fit), sequence 1 at 0..7; both rows of
    # sequence 1 stay untouched by sequence 0's overflow
    start = torch.tensor([28, 0], dtype=torch.int64, device="cuda")
    flags = torch.zeros(B, 8, dtype=torch.uint8, device="cuda")
    flags[0, 1] = 1  # sink at 29
    flags[0, 2] = 1  # second sink: sidecar (1) full -> stays quantized
    flags[0, 6] = 1  # past capacity: ignored
    layer.append_device(k, v, start, flags)
    torch.cuda.synchronize()
    a = cache_host(layer)
    kc, km, vc, vm = oracle.quantize_kv_rows(k[1].cpu().numpy(), v[1].cpu().numpy(), 8, 128, 4, perm)
    assert np.array_equal(a["k_codes"][1, :8].view(np.uint32), kc)
    assert np.array_equal(a["v_meta"][1, :8].view(np.uint32), vm)
    kc0, km0, _, _ = oracle.quantize_kv_rows(k[0].cpu().numpy(), v[0].cpu().numpy(), 8, 128, 4, perm)
    assert np.array_equal(a["k_codes"][0, 28].view(np.uint32), kc0[0])
    assert not a["k_codes"][0, 29].any()                                   # the sink
    assert np.array_equal(a["k_codes"][0, 30].view(np.uint32), kc0[2])    # sidecar full: quantized
    assert int(a["sink_count"][0]) == 1 and int(a["sink_pos"][0, 0]) == 29
    mask = a["sink_mask"][0].view(np.uint32)[0]
    assert (mask >> 29) & 1 and not (mask >> 30) & 1


def test_foreign_plan_yields_nan():
    """A plan built for another layer width makes decode emit NaN."""
    w = small_workload(8, 8, 4)
    layer, perm = build_layer(w, 1, 64, seed=52)
    k, v = WL.make_kv(w, 52, 1, 40)
    layer.append(k, v)
    q = WL.make_q(w, 52, 1)
    good = layer.decode(q)
    assert torch.isfinite(good).all()
    w2 = small_workload(16, 16, 4)
    other, _ = build_layer(w2, 1, 64, seed=53)
    layer.plan = other.plan  # C = 2048 plan on a C = 1024 layer
    bad = layer.decode(q)
    assert torch.isnan(bad).all()


def test_rotate_keys_beyond_grid_y_limit(oracle):
    w = small_workload(8, 8, 4)
    cfg = P.LayerConfig(batch=1, num_q_heads=8, num_kv_heads=8, heads_per_group=4)
    rows = 70000
    k, _ = WL.make_kv(w, 54, 1, rows)
    got = P.rotate_keys(cfg, k[0])
    torch.cuda.synchronize()
    sel = np.array([0, 1, 65534, 65535, 65536, rows - 1])
    want = oracle.rotate_rows(k[0, sel].float().cpu().numpy(), 128, 4, 8)
    assert np.array_equal(got[sel].cpu().numpy(), want)
    perm, _ = P.calibrate_reorder_device(cfg, k[0])
    assert np.array_equal(np.sort(perm), np.arange(1024))
