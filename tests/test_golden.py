"""Pin the oracle on fixtures generated from the unmodified reference
(tests/golden/make_golden.py).  Runs everywhere, including the GPU box where
/root/reference is absent.  CPU only."""
import os

import numpy as np
import pytest

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(G, name))


def test_golden_quant_group(oracle):
    f = load("quant_group_e4m3.npz")
    for x, sc, z, packed in zip(f["x"], f["scale_e4m3"], f["zero"], f["packed"]):
        s, zz, codes, code = oracle.quantize_group(x, 2, oracle.SCALE_E4M3_CEIL)
        assert code == sc and zz == z
        assert np.array_equal(oracle.pack_codes(codes, 2), packed)


def test_golden_fwht(oracle):
    f = load("fwht512.npz")
    for x, y in zip(f["x"], f["y"]):
        assert np.array_equal(oracle.fwht(x), y)


def test_golden_calibrate(oracle):
    f = load("calibrate.npz")
    perm, inv = oracle.calibrate_reorder(f["rows"])
    assert np.array_equal(perm, f["perm"]) and np.array_equal(inv, f["inverse"])


def test_golden_rope(oracle):
    f = load("rope.npz")
    assert np.array_equal(oracle.apply_rope_rows(f["x"], 2, 128, 10000.0, f["pos"]), f["y10k"])
    assert np.array_equal(oracle.apply_rope_rows(f["x"], 2, 128, 500000.0, f["pos"]), f["y500k"])


def test_golden_quantize_kv(oracle):
    f = load("quantize_kv_e4m3.npz")
    h, d, g = int(f["h"]), int(f["d"]), int(f["g"])
    kc, km, vc, vm = oracle.quantize_kv_rows(f["k"], f["v"], h, d, g, f["perm"], oracle.SCALE_E4M3_CEIL)
    assert np.array_equal(kc, f["k_codes"]) and np.array_equal(vc, f["v_codes"])
    dec = np.vectorize(lambda s: oracle.e4m3_decode(int(s)))
    assert np.array_equal((km & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float32), dec(f["k_scale"]))
    assert np.array_equal((km >> 16).astype(np.uint16).view(np.float16).astype(np.float32), f["k_zero"].astype(np.float32))
    assert np.array_equal((vm & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float32), dec(f["v_scale"]))
    assert np.array_equal((vm >> 16).astype(np.uint16).view(np.float16).astype(np.float32), f["v_zero"].astype(np.float32))


def test_golden_decode_step(oracle):
    f = load("decode_step.npz")
    h, d, g = int(f["h"]), int(f["d"]), int(f["g"])
    k, v, x, sink, perm = f["k"], f["v"], f["x"], f["sink"], f["perm"]
    K = np.concatenate([k, x[None]])
    V = np.concatenate([v, x[None]])
    S = np.concatenate([sink, [0]]).astype(np.uint8)
    kc, km, vc, vm = oracle.quantize_kv_rows(K, V, h, d, g, perm, oracle.SCALE_E4M3_CEIL)
    got = oracle.decode_attention(kc, km, vc, vm, S, K, V, x, h, h, d, g, perm, float(f["base"])).reshape(-1)
    want = f["out"]
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-4


def test_golden_sinks(oracle):
    f = load("sinks.npz")
    assert np.array_equal(oracle.detect_sinks(f["hidden"]), f["flags"])
