"""Layers of different widths in one process: per-kernel launch attributes
(dynamic shared-memory limits) must be set for each launch's own size, so a
narrower layer launched in between cannot break a wider one."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2501_16383_b200 as P  # noqa: E402


def layer(heads, g=4):
    cfg = P.LayerConfig(batch=2, num_q_heads=heads, num_kv_heads=heads, heads_per_group=g, max_tokens=64,
                        max_sinks=2)
    perm = np.random.default_rng(heads).permutation(heads * 128).astype(np.int32)
    return P.RotateKVLayer(cfg, perm)


def step(lay, n=8):
    c = lay.cfg.channels
    k = torch.randn(2, n, c, device="cuda").to(torch.float16)
    lay.append(k, k)
    q = torch.randn(2, lay.cfg.num_q_heads, 128, device="cuda").to(torch.float16)
    out = lay.decode(q)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()


def test_wide_narrow_wide():
    wide, narrow = layer(40), layer(32)
    step(wide)
    step(narrow)
    step(wide)
    step(narrow)
