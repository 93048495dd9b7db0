"""GPU sink detection (csrc/sink_detect.cu) vs the oracle's
restatement of detect_massive_activations (proj/src/sink.cpp:14-45): the
flags and the median must be identical (the median is an exact radix select,
the threshold compare is exact in fp32)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402


def run(x, rel=50.0, floor=0.0):
    flags, med = P.detect_massive_activations_device(torch.from_numpy(x).cuda(), rel, floor, return_median=True)
    return flags.cpu().numpy(), float(med.item())


def expected_median(x):
    m = np.sort(np.abs(x).reshape(-1))
    return float(m[m.size // 2])


@pytest.mark.parametrize("b,s,h,seed", [(1, 1, 1, 0), (1, 7, 5, 1), (2, 33, 64, 2), (3, 128, 96, 3),
                                        (1, 4096, 512, 4), (2, 257, 1023, 5)])
def test_random_spikes(oracle, b, s, h, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((b, s, h)).astype(np.float32)
    for t in rng.choice(s, size=min(3, s), replace=False):
        x[rng.integers(b), t, rng.integers(h)] = rng.choice([-1, 1]) * rng.uniform(60, 200)
    flags, med = run(x)
    assert med == expected_median(x)
    assert np.array_equal(flags, oracle.detect_sinks(x))


def test_workload_hidden_states(oracle):
    w = WL.CONFIGS[3]
    x = WL.hidden_with_sinks(w, 11, 2048)
    flags, _ = run(x)
    want = oracle.detect_sinks(x)
    assert np.array_equal(flags, want)
    assert np.array_equal(flags, P.detect_massive_activations(x))
    assert want.sum() >= 3  # token 0 + the seeded delimiters


def test_boundaries_and_ties(oracle):
    # many exact ties around the median, values exactly at the threshold,
    # negative zero, subnormals, and an abs_floor that dominates
    x = np.full((2, 64, 32), 0.5, np.float32)
    x[:, :, :16] = 1.0         # 2048 values below 1.0, so the median (index n/2) is 1.0
    x[0, 5, 3] = 50.0          # == 50 * median: not a sink (strict >)
    x[1, 9, 4] = np.nextafter(np.float32(50.0), np.float32(100.0))  # just above
    x[0, 12, 20] = -np.float32(0.0)
    x[1, 20, 21] = np.float32(1e-45)
    flags, med = run(x)
    assert med == expected_median(x) == 1.0
    assert np.array_equal(flags, oracle.detect_sinks(x))
    assert np.flatnonzero(flags).tolist() == [0, 9]
    flags2, _ = run(x, rel=2.0, floor=60.0)
    assert np.array_equal(flags2, oracle.detect_sinks(x, 2.0, 60.0))
    assert np.flatnonzero(flags2).tolist() == [0]


def test_rejects_bad_arguments():
    x = torch.zeros(1, 4, 8, device="cuda")
    with pytest.raises(ValueError, match="rel_threshold"):
        P.detect_massive_activations_device(x, rel_threshold=1.0)
    with pytest.raises(ValueError, match="float32"):
        P.detect_massive_activations_device(x.half())


def test_flags_feed_quantize(oracle):
    """Device flags -> rkv_quantize_kv sink routing without a host round trip."""
    w = WL.Workload("t", 1, 8, 8, 0, 4, 10000.0, 4, (10.0, 30.0))
    B, T = 2, 64
    cfg = P.LayerConfig(batch=B, num_q_heads=8, num_kv_heads=8, heads_per_group=4, max_tokens=T, max_sinks=8)
    perm = WL.calibration_perm(w, 3)
    layer = P.RotateKVLayer(cfg, perm)
    hid = np.random.default_rng(4).standard_normal((B, T, 256)).astype(np.float32)
    hid[1, 17, 5] = 500.0
    flags = P.detect_massive_activations_device(torch.from_numpy(hid).cuda())
    k, v = WL.make_kv(w, 5, B, T)
    start = torch.zeros(B, dtype=torch.int64, device="cuda")
    layer.append_device(k, v, start, flags.unsqueeze(0).expand(B, T).contiguous())
    torch.cuda.synchronize()
    a = layer.arrays()
    assert a["sink_count"].cpu().tolist() == [2, 2]
    assert a["sink_pos"].cpu().numpy()[:, :2].tolist() == [[0, 17], [0, 17]]
