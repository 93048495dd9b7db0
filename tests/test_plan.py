"""The per-layer decode plan (csrc/rkv_plan.cu): which packed word each decode
thread un-reorders, chosen to minimise shared-memory bank conflicts of the
scatter.  Host-only, CPU.

Checked: the word -> position map is a permutation; code e of the word at
position wp is stored at the K-tile position of its natural channel
perm[16w+e] (rkv_layout.h, padded rows); and the optimised assignment's
bank-conflict cost is well below taking words in order."""
import numpy as np
import pytest

import paper_2501_16383_b200 as P

HEADER = 16


def knat_pos(N, c):
    L = 16 if N >= 256 else 8
    R = N // L
    g, i = c // N, c % N
    return g * L * (R + 1) + (i // R) * (R + 1) + (i % R)


def cost_of(cls, omega):
    tot = 0
    for k in range(len(omega) // 16):
        words = omega[16 * k:16 * k + 16]
        for e in range(16):
            tot += np.bincount(cls[words, e], minlength=16).max()
    return tot


@pytest.mark.parametrize("hq,hkv,g,seed", [(40, 40, 4, 0), (32, 32, 4, 1), (32, 8, 2, 2), (8, 8, 4, 3), (4, 4, 1, 4)])
def test_plan_is_a_valid_scatter(hq, hkv, g, seed):
    cfg = P.LayerConfig(batch=1, num_q_heads=hq, num_kv_heads=hkv, heads_per_group=g)
    C = hkv * 128
    N = 128 * g
    perm = np.random.default_rng(seed).permutation(C).astype(np.int32)
    words, cost = P.layer_plan_build(cfg, perm)
    assert int(words[0]) == 0x504B5652 and int(words[2]) == N and int(words[4]) == C
    W = C // 16
    omega = words[HEADER:HEADER + W].astype(np.int64)
    addr = words[HEADER + W:HEADER + W + 16 * W].reshape(4, W, 4)
    assert sorted(omega.tolist()) == list(range(W))
    for wp in range(W):
        w = omega[wp]
        for e in range(16):
            assert addr[e // 4, wp, e % 4] == knat_pos(N, int(perm[16 * w + e])) * 8
    cls = np.array([knat_pos(N, int(c)) % 16 for c in perm]).reshape(W, 16)
    assert cost == cost_of(cls, omega)
    if W >= 32:  # more than one half-warp group: the assignment must beat the identity
        assert cost < 0.85 * cost_of(cls, np.arange(W))


def test_plan_rejects_non_permutation():
    cfg = P.LayerConfig(batch=1, num_q_heads=8, num_kv_heads=8, heads_per_group=4)
    with pytest.raises(ValueError, match="permutation"):
        P.layer_plan_build(cfg, np.zeros(1024, np.int32))
