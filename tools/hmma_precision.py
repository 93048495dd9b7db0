"""Numerical check of a tensor-core (mma.sync fp16) decode formulation before
building it: emulates fp16 rounding of the dequantized K (X), of the half-way
FWHT result (Y), and of the V weights p*s, and compares the decode output with
the exact (float64) decode over the same 2-bit cache.

    python tools/hmma_precision.py [cfg] [tokens]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402


def fwht_bits(x, bits):
    """Unnormalised Walsh-Hadamard over the given index bits of the last axis."""
    y = x.copy()
    for b in bits:
        h = 1 << b
        n = y.shape[-1]
        idx = np.arange(n)
        lo = idx[(idx & h) == 0]
        a, c = y[..., lo].copy(), y[..., lo + h].copy()
        y[..., lo], y[..., lo + h] = a + c, a - c
    return y


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    w = WL.CONFIGS[cfg]
    C, G, d = w.channels, w.heads_per_group, 128
    N = G * d
    Hq, Hkv = w.num_q_heads, w.num_kv_heads
    import torch

    k, v = WL.make_kv(w, 42 + cfg, 1, T, device="cpu")
    kc, _ = WL.make_kv(w, 42 + cfg + 100, 1, 256, device="cpu")
    rk = oracle.rotate_rows(kc[0].float().numpy(), d, G, Hkv)
    perm, _ = oracle.calibrate_reorder(rk, oracle.STAT_MEAN_ABS)
    kq, kmq, vq, vmq = oracle.quantize_kv_rows(k[0].numpy(), v[0].numpy(), Hkv, d, G, perm)
    q = WL.make_q(w, 42 + cfg, 1, device="cpu")[0].float().numpy().astype(np.float64)

    def deq(codes, meta):
        c = ((codes[:, :, None] >> (2 * np.arange(16))) & 3).reshape(T, C).astype(np.float64)
        s = np.array([oracle.half_to_float(int(m) & 0xFFFF) for m in meta.ravel()]).reshape(T, C // 128)
        z = np.array([oracle.half_to_float(int(m) >> 16) for m in meta.ravel()]).reshape(T, C // 128)
        return c, np.repeat(s, 128, 1), np.repeat(z, 128, 1)

    ck, sk, zk = deq(kq, kmq)
    cv, sv, zv = deq(vq, vmq)
    uslot = sk * (ck - zk)                       # exact in fp32
    inv = np.argsort(perm)
    unat = uslot[:, inv]                         # slot j -> channel perm[j]

    pos = np.arange(T, dtype=np.float64)
    theta = w.rope_base ** (-2.0 * np.arange(64) / 128.0)
    ang = pos[:, None] * theta[None, :]
    cos, sin = np.cos(ang), np.sin(ang)

    def rope(x):  # [T, heads, 128]
        a, b = x[..., :64], x[..., 64:]
        return np.concatenate([a * cos[:, None] - b * sin[:, None], a * sin[:, None] + b * cos[:, None]], -1)

    qa, qb = q[:, :64], q[:, 64:]
    cq, sq = np.cos((T - 1) * theta), np.sin((T - 1) * theta)
    qr = np.concatenate([qa * cq - qb * sq, qa * sq + qb * cq], -1)

    def decode(knat, vw_round):
        kr = rope(knat.reshape(T, Hkv, d))
        rep = Hq // Hkv
        logits = np.einsum("hd,thd->ht", qr, np.repeat(kr, rep, 1)) / np.sqrt(d)
        m = logits.max(1, keepdims=True)
        p = np.exp(logits - m)
        l = p.sum(1)
        vrot = (sv * (cv - zv)).reshape(T, Hkv, d)
        if vw_round is None:
            o = np.einsum("ht,thd->hd", p, np.repeat(vrot, rep, 1))
        else:  # weights p*s rounded to fp16 (hi, optionally + lo), codes exact, z-term exact
            svh = sv.reshape(T, Hkv, d)[:, :, 0]
            zvh = zv.reshape(T, Hkv, d)[:, :, 0]
            ps = p * np.repeat(svh, rep, 1).T
            hi = ps.astype(np.float16).astype(np.float64)
            wgt = hi if vw_round == "hi" else hi + (ps - hi).astype(np.float16).astype(np.float64)
            cvh = np.repeat(cv.reshape(T, Hkv, d), rep, 1)
            # the zero point uses the same rounded weights (consistent, as the kernel does)
            o = np.einsum("ht,thd->hd", wgt, cvh) - (wgt * np.repeat(zvh, rep, 1).T).sum(1)[:, None]
        o = fwht_bits(o, range(7)) / np.sqrt(128.0)
        return o / l[:, None]

    exact_k = fwht_bits(unat.reshape(T, C // N, N), range(int(np.log2(N)))).reshape(T, C) / np.sqrt(N)
    ref = decode(exact_k, None)

    lb = int(np.log2(N))
    other = [b for b in range(lb) if b != 6]
    f1, f2 = other[:4], other[4:]
    x16 = unat.astype(np.float32).astype(np.float16).astype(np.float64)
    for label, xin, yround, vr in [
        ("X fp16, Y fp16, V hi", x16, True, "hi"),
        ("X fp16, Y fp16, V hi+lo", x16, True, "hilo"),
        ("X fp16, Y hi+lo, V hi+lo", x16, "hilo", "hilo"),
        ("X fp16, Y hi+lo, V hi", x16, "hilo", "hi"),
        ("X exact, Y fp16, V hi+lo", unat, True, "hilo"),
    ]:
        y = fwht_bits(xin.reshape(T, C // N, N), f1)
        if yround is True:
            y = y.astype(np.float32).astype(np.float16).astype(np.float64)
        elif yround == "hilo":
            yh = y.astype(np.float32).astype(np.float16).astype(np.float64)
            y = yh + (y - yh).astype(np.float32).astype(np.float16).astype(np.float64)
        z = fwht_bits(y, f2 + [6]).reshape(T, C) / np.sqrt(N)
        out = decode(z, vr)
        err = np.abs(out - ref).max() / np.abs(ref).max()
        cosv = (out * ref).sum() / np.linalg.norm(out) / np.linalg.norm(ref)
        print(f"cfg{cfg} T={T} {label:28s}: max rel err {err:.2e}  cosine {cosv:.8f}")


if __name__ == "__main__":
    main()
