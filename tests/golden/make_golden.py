"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

Run in a container that has /root/reference (so oracle/_ref can be built):
    python tests/golden/make_golden.py
Every expected output below is produced by the reference's own functions via
oracle/ref_adapter.cpp; the inputs are seeded synthetic data.  The fixtures
let tests/test_golden.py pin the oracle where the reference is absent (the
GPU box).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def groups(rng, n):
    xs = []
    for i in range(n):
        scale = rng.choice([1e-6, 1e-3, 0.1, 1.0, 7.0, 100.0, 3000.0])
        x = (rng.standard_normal(128) * scale).astype(np.float32)
        if i % 3 == 0:
            lo, hi = float(x.min()), float(x.max())
            s = (hi - lo) / 3.0
            ks = rng.integers(-3, 4, 16)
            x[rng.integers(0, 128, 16)] = ((ks - 0.5) * s).astype(np.float32)
            x = np.clip(x, lo, hi).astype(np.float32)
        if i % 7 == 0:
            x[:] = np.float32(scale)
        xs.append(x)
    return np.stack(xs)


def main():
    O.build(ref=True)
    rng = np.random.default_rng(20250127)
    save = lambda name, **kw: np.savez_compressed(os.path.join(HERE, name), **kw)

    x = groups(rng, 256)
    sc, z, packed = [], [], []
    for g in x:
        a, b, _, p = O.ref_quantize_group(g, 2, 128)
        sc.append(a), z.append(b), packed.append(p)
    save("quant_group_e4m3.npz", x=x, scale_e4m3=np.uint8(sc), zero=np.uint8(z), packed=np.stack(packed))

    v = (rng.standard_normal((8, 512)) * 20).astype(np.float32)
    save("fwht512.npz", x=v, y=np.stack([O.fwht(r, impl="ref") for r in v]))

    rows = rng.standard_normal((32, 1024)).astype(np.float32)
    rows[:, rng.integers(0, 1024, 12)] *= 25
    perm, inv = O.calibrate_reorder(rows, impl="ref")
    save("calibrate.npz", rows=rows, perm=perm, inverse=inv)

    r = rng.standard_normal((4, 256)).astype(np.float32)
    pos = np.array([0, 5, 4095, 32767], np.int64)
    save("rope.npz", x=r, pos=pos, y10k=O.apply_rope_rows(r, 2, 128, 10000.0, pos, impl="ref"),
         y500k=O.apply_rope_rows(r, 2, 128, 500000.0, pos, impl="ref"))

    h, d, g = 8, 128, 4
    c = h * d
    k = rng.standard_normal((8, c)).astype(np.float16)
    k[:, rng.integers(0, c, 16)] *= np.float16(20)
    vv = rng.standard_normal((8, c)).astype(np.float16)
    perm = rng.permutation(c).astype(np.int32)
    kc, ks, kz, vc, vs, vz = O.ref_quantize_kv_rows(k.astype(np.float32), vv.astype(np.float32), h, d, g, perm)
    save("quantize_kv_e4m3.npz", k=k, v=vv, perm=perm, h=h, d=d, g=g, k_codes=kc, k_scale=ks, k_zero=kz,
         v_codes=vc, v_scale=vs, v_zero=vz)

    T = 24
    k = rng.standard_normal((T, c)).astype(np.float16)
    k[:, rng.integers(0, c, 16)] *= np.float16(15)
    vv = rng.standard_normal((T, c)).astype(np.float16)
    xq = rng.standard_normal(c).astype(np.float16)
    sink = np.zeros(T, np.uint8)
    sink[[0, 9]] = 1
    out = O.ref_decode_step(k.astype(np.float32), vv.astype(np.float32), sink, perm, xq.astype(np.float32), h, d, g, 10000.0)
    save("decode_step.npz", k=k, v=vv, x=xq, sink=sink, perm=perm, h=h, d=d, g=g, base=10000.0, out=out)

    hid = rng.standard_normal((1, 64, 256)).astype(np.float32)
    hid[0, 0, 17] = 100.0
    hid[0, 41, 3] = -120.0
    save("sinks.npz", hidden=hid, flags=O.detect_sinks(hid, impl="ref"))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
