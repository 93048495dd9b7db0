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


def mma_pos(N, c):
    """Byte offset of channel c in the tensor-core kernel's token-pair row (rkv_layout.h mma_pos)."""
    g, i = c // N, c % N
    k = i & 15
    n = ((i >> 4) & 1) | (((i >> 5) & 1) << 1) | (((i >> 7) & 1) << 2)
    jc = (((i >> 8) & 1) | (((i >> 6) & 1) << 1)) if N == 512 else ((i >> 6) & 1)
    lane = 4 * n + ((k >> 1) & 3)
    nj = N // 128
    swz = ((lane >> 1) & 3) if N == 512 else ((lane >> 2) & 1)
    return g * N * 4 + lane * nj * 16 + (jc ^ swz) * 16 + ((k >> 3) * 2 + (k & 1)) * 4


def cost_of(cls, omega, gs=16):
    tot = 0
    for k in range((len(omega) + gs - 1) // gs):  # the last store group may be partial
        words = omega[gs * k:gs * k + gs]
        for e in range(16):
            tot += np.bincount(cls[words, e], minlength=gs).max()
    return tot


def test_mma_positions_are_a_bijection():
    for N, C in [(512, 5120), (512, 4096), (256, 1024)]:
        pos = sorted(mma_pos(N, c) for c in range(C))
        assert pos == list(range(0, 4 * C, 4))


@pytest.mark.parametrize("hq,hkv,g,seed", [(40, 40, 4, 0), (32, 32, 4, 1), (32, 8, 2, 2), (8, 8, 4, 3), (4, 4, 1, 4),
                                           (8, 8, 1, 5), (8, 8, 2, 6), (40, 40, 1, 7),
                                           # GQA at other ratios and widths; 80 and 48 words leave a
                                           # partial store group
                                           (40, 10, 2, 8), (24, 6, 2, 9), (64, 16, 4, 10), (16, 8, 2, 11),
                                           (128, 16, 2, 12), (24, 8, 4, 13)])
def test_plan_is_a_valid_scatter(hq, hkv, g, seed):
    cfg = P.LayerConfig(batch=1, num_q_heads=hq, num_kv_heads=hkv, heads_per_group=g)
    C = hkv * 128
    perm = np.random.default_rng(seed).permutation(C).astype(np.int32)
    words, cost = P.layer_plan_build(cfg, perm)
    mma = int(words[7]) == 1  # PH_KIND: tensor-core decode layout
    # tensor-core layouts tile 512 channels (MHA, G = 4, 2 or 1 heads per rotation
    # group) or 256 (GQA, G = 2); the CUDA-core layout follows the rotation group
    gqa = g in (1, 2, 4) and hq >= 2 * hkv and C % (128 * max(g, 2)) == 0 and C // 256 <= 8
    N = (256 if gqa else 512) if mma else 128 * g
    assert mma == (gqa or (hq == hkv and C % 512 == 0))
    assert int(words[0]) == 0x504B5652 and int(words[2]) == N and int(words[4]) == C
    W = C // 16
    omega = words[HEADER:HEADER + W].astype(np.int64)
    addr = words[HEADER + W:HEADER + W + 16 * W].reshape(4, W, 4)
    assert sorted(omega.tolist()) == list(range(W))
    pos = (lambda c: mma_pos(N, c)) if mma else (lambda c: knat_pos(N, c) * 8)
    for wp in range(W):
        w = omega[wp]
        for e in range(16):
            assert addr[e // 4, wp, e % 4] == pos(int(perm[16 * w + e]))
    gs = 32 if mma else 16
    cls = np.array([(pos(int(c)) >> 2) % 32 if mma else (pos(int(c)) >> 3) % 16 for c in perm]).reshape(W, 16)
    assert cost == cost_of(cls, omega, gs)
    if W >= 2 * gs:  # more than one store group: the assignment must beat the identity
        ident = cost_of(cls, np.arange(W), gs)
        assert cost < (0.85 if W >= 4 * gs else 0.95) * ident


def test_plan_rejects_non_permutation():
    cfg = P.LayerConfig(batch=1, num_q_heads=8, num_kv_heads=8, heads_per_group=4)
    with pytest.raises(ValueError, match="permutation"):
        P.layer_plan_build(cfg, np.zeros(1024, np.int32))
