"""GPU calibration statistics (rkv_calibrate_reorder_device):
raw fp16 K rows -> rotate_rows -> per-channel double statistic -> stable
argsort (proj/src/pipeline.cpp:101-109, proj/src/reorder.cpp:91-110).  The
permutation must be identical to the oracle's calibrate_reorder on the
oracle's rotation of the same rows, for both statistics (the reference's
signed sum and the north star's mean |K|), MHA/GQA shapes and G = 1, 2, 4."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402


@pytest.mark.parametrize("hq,hkv,g,rows,seed", [(8, 8, 4, 256, 0), (40, 40, 4, 256, 1), (32, 8, 2, 256, 2),
                                                (4, 4, 1, 33, 3), (16, 16, 4, 1, 4), (32, 32, 4, 512, 5)])
@pytest.mark.parametrize("stat", [P.STAT_SUM, P.STAT_MEAN_ABS])
def test_device_calibration_matches_oracle(oracle, hq, hkv, g, rows, seed, stat):
    C = hkv * 128
    cfg = P.LayerConfig(batch=1, num_q_heads=hq, num_kv_heads=hkv, heads_per_group=g, max_tokens=max(rows, 2))
    w = WL.Workload("calib", 1, hq, hkv, rows, g, 10000.0, 4, (10.0, 30.0))
    k, _ = WL.make_kv(w, seed, 1, rows, device="cuda")
    k = k.reshape(rows, C)
    perm, inv = P.calibrate_reorder_device(cfg, k, stat)
    rk = oracle.rotate_rows(k.cpu().numpy().astype(np.float32), 128, g, hkv)
    want, _ = oracle.calibrate_reorder(rk, stat)
    assert np.array_equal(perm, want)
    assert np.array_equal(inv[perm], np.arange(C))
    # and the host C-ABI path on the device rotation
    hp, _ = P.calibrate_reorder(P.rotate_keys(cfg, k).cpu().numpy(), stat)
    assert np.array_equal(hp, want)


def test_ties_keep_channel_order():
    """Constant (all-zero) keys: every statistic ties, stable sort keeps 0..C-1."""
    cfg = P.LayerConfig(batch=1, num_q_heads=8, num_kv_heads=8, heads_per_group=4, max_tokens=16)
    k = torch.zeros(16, 1024, dtype=torch.float16, device="cuda")
    perm, _ = P.calibrate_reorder_device(cfg, k, P.STAT_SUM)
    assert np.array_equal(perm, np.arange(1024))


def test_rejects_bad_arguments():
    cfg = P.LayerConfig(batch=1, num_q_heads=8, num_kv_heads=8, heads_per_group=4, max_tokens=16)
    k = torch.zeros(16, 1024, dtype=torch.float16, device="cuda")
    with pytest.raises(ValueError, match="statistic"):
        P.calibrate_reorder_device(cfg, k, 7)
    with pytest.raises(ValueError, match="empty"):
        P.calibrate_reorder_device(cfg, k[:0], P.STAT_SUM)
