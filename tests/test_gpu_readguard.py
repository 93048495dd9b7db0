"""Out-of-bounds reads of the cache fault instead of passing silently.

The carved cache is placed flush against an unmapped hole in the virtual
address space (driver VMM: cuMemAddressReserve / cuMemCreate / cuMemMap), once
with its last byte on the last mapped byte and once with its first byte on the
first mapped byte.  Batch and max_tokens are chosen so the last sequence's
sink-mask row (the last carved array) ends exactly at the cache's end, with no
256-byte padding behind it.  Every kernel family then runs over a full cache:
a read one word past the last sequence's rows or before the first array is an
illegal-address fault.  The appended K/V rows (an odd token count), the
queries, the fused-frame rows, the calibration keys and the sink-detection
hidden states are placed the same way.  Each placement runs in a child process so a fault
cannot poison the other GPU tests; results must also equal the same calls on
an ordinary allocation.  A positive control checks that the neighbouring
bytes of such a mapping really are unreadable.
"""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (hq, hkv, G, batch, max_tokens): B * ceil(T / 32) is a multiple of 64
CASES = [
    (8, 8, 4, 4, 500),     # MHA tensor-core kernel
    (8, 8, 1, 2, 1000),    # MHA at G = 1
    (16, 4, 2, 4, 500),    # GQA 4:1, G = 2
    (16, 4, 4, 2, 1000),   # GQA 4:1, G = 4 (half-group pairs)
    (16, 16, 8, 8, 250),   # tiled generic kernels
    (40, 40, 4, 4, 500),   # C = 5120, warp-independent V quantize
]


def _child(at):
    import ctypes as C

    import numpy as np
    from cuda.bindings import driver as cu

    sys.path.insert(0, ROOT)
    import paper_2501_16383_b200 as P  # noqa: F401
    from paper_2501_16383_b200 import rotatekv as RK
    from paper_2501_16383_b200 import workload as WL
    from tests.test_gpu_parity import build_layer, small_workload

    def ok(r):
        assert r[0] == cu.CUresult.CUDA_SUCCESS, r[0]
        return r[1] if len(r) == 2 else r[1:]

    torch.cuda.init()
    torch.empty(1, device="cuda")
    ok((cu.cuInit(0)[0], None))
    dev = torch.cuda.current_device()
    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = dev
    gran = ok(cu.cuMemGetAllocationGranularity(
        prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))

    acc = cu.CUmemAccessDesc()
    acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = dev
    acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    maps = []

    def edge_alloc(nbytes):
        """nbytes flush against an unmapped hole at the `at` end"""
        size = (nbytes + gran - 1) // gran * gran
        va = int(ok(cu.cuMemAddressReserve(size + 2 * gran, 0, 0, 0)))
        h = ok(cu.cuMemCreate(size, prop, 0))
        mapped = va + gran
        ok((cu.cuMemMap(mapped, size, 0, h, 0)[0], None))
        ok((cu.cuMemSetAccess(mapped, size, [acc], 1)[0], None))
        maps.append((va, h, mapped, size))
        return mapped + size - nbytes if at == "end" else mapped

    class Raw:  # a torch view of raw device memory (no copy)
        def __init__(self, ptr, shape, typestr):
            self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                             "version": 3, "strides": None}

    def edge_like(t):
        ts = {torch.float16: "<f2", torch.float32: "<f4"}[t.dtype]
        e = torch.as_tensor(Raw(edge_alloc(t.numel() * t.element_size()), t.shape, ts), device="cuda")
        e.copy_(t)
        return e

    def carve_edge(layer):
        """re-carve the layer's cache at the hole (its arrays() views included)"""
        nbytes = RK.lib().rkv_cache_bytes(C.byref(layer._desc))
        assert nbytes % 256 == 0
        base = edge_alloc(nbytes)
        RK._check(RK.lib().rkv_cache_carve(C.byref(layer._desc), base, nbytes, C.byref(layer._view)))
        layer._buf = torch.as_tensor(Raw(base, (nbytes,), "|u1"), device="cuda")
        layer._base = base
        layer.reset()

    def release():
        torch.cuda.synchronize()
        for va, h, mapped, size in maps:
            ok((cu.cuMemUnmap(mapped, size)[0], None))
            ok((cu.cuMemRelease(h)[0], None))
            ok((cu.cuMemAddressFree(va, size + 2 * gran)[0], None))
        maps.clear()

    for hq, hkv, g, B, T in CASES:
        w = small_workload(hq, hkv, g)
        plain, perm = build_layer(w, B, T, seed=71, max_sinks=2)
        edge, _ = build_layer(w, B, T, seed=71, max_sinks=2, perm=perm)
        carve_edge(edge)

        n = T - 1  # an odd append: the last token pair has one row
        k, v = WL.make_kv(w, 71, B, n)
        flags = torch.zeros(B, n, dtype=torch.uint8)
        flags[:, 0] = 1
        flags[B - 1, n - 1] = 1
        plain.append(k, v, flags)
        edge.append(edge_like(k), edge_like(v), flags)  # the new rows flush against a hole too
        q = WL.make_q(w, 71, B)
        qe = edge_like(q)
        ragged = np.maximum(1, n - 45 * np.arange(B, dtype=np.int64))
        for lens in (None, ragged):
            a, b = plain.decode(q, seq_len=lens), edge.decode(qe, seq_len=lens)
            torch.cuda.synchronize()
            assert torch.equal(a, b), (hq, hkv, g, "decode")
        if g != 8:
            qp = torch.randn(B, 64, hq, 128, generator=torch.Generator().manual_seed(9)).half().cuda()
            a, b = plain.prefill_attention(qp), edge.prefill_attention(edge_like(qp))
            torch.cuda.synchronize()
            assert torch.equal(a, b), (hq, hkv, g, "prefill")
        data = edge.serialize(B - 1)
        assert data == plain.serialize(B - 1), (hq, hkv, g, "export")
        del edge, qe
        release()
        print(f"ok {at} {hq}/{hkv} G={g} B={B} T={T}", flush=True)

    # the other readers of caller buffers: the fused-frame append (fp32 and
    # fp16 rows, odd count), device calibration and device sink detection
    w = small_workload(40, 40, 4)
    B, T, n = 4, 500, 499
    plain, perm = build_layer(w, B, T, seed=72, max_sinks=2)
    edge, _ = build_layer(w, B, T, seed=72, max_sinks=2, perm=perm)
    carve_edge(edge)
    gen = torch.Generator().manual_seed(4)
    rows = torch.randn(B, n, 5120, generator=gen).cuda()
    flags = torch.zeros(B, n, dtype=torch.uint8)
    flags[:, 0] = 1
    for lo, hi, dt in ((0, 250, torch.float32), (250, n, torch.float16)):
        kr, vr = rows[:, lo:hi].to(dt).contiguous(), (rows[:, lo:hi] * 0.5).to(dt).contiguous()
        plain.append_fused(kr, vr, flags[:, lo:hi])
        edge.append_fused(edge_like(kr), edge_like(vr), flags[:, lo:hi])
    torch.cuda.synchronize()
    ta, tb = plain.arrays(), edge.arrays()
    for name in ("k_codes", "v_codes", "k_meta", "v_meta"):
        assert torch.equal(ta[name][:, :n], tb[name][:, :n]), ("fused append", name)
    kcal = torch.randn(1001, 5120, generator=gen).half().cuda()
    assert np.array_equal(P.calibrate_reorder_device(plain.cfg, kcal)[0],
                          P.calibrate_reorder_device(plain.cfg, edge_like(kcal))[0]), "calibration"
    hidden = torch.randn(2, 333, 512, generator=gen).cuda()
    hidden[:, 7, 3] = 400.0
    fa, fb = P.detect_massive_activations_device(hidden), P.detect_massive_activations_device(edge_like(hidden))
    assert torch.equal(fa, fb) and int(fa[7]) == 1, "sink detection"
    del edge
    release()
    print(f"ok {at} fused append / calibration / sink detection", flush=True)

    # positive control: the byte just outside a mapped region is not readable
    va = int(ok(cu.cuMemAddressReserve(3 * gran, 0, 0, 0)))
    h = ok(cu.cuMemCreate(gran, prop, 0))
    ok((cu.cuMemMap(va + gran, gran, 0, h, 0)[0], None))
    ok((cu.cuMemSetAccess(va + gran, gran, [acc], 1)[0], None))
    host = np.zeros(4, np.uint8)
    assert cu.cuMemcpyDtoH(host, va + gran + gran - 4, 4)[0] == cu.CUresult.CUDA_SUCCESS
    probe = va + gran + gran if at == "end" else va + gran - 4
    r = cu.cuMemcpyDtoH(host, probe, 4)[0]
    assert r != cu.CUresult.CUDA_SUCCESS, "unmapped neighbour was readable"
    print(f"control {at}: {r}", flush=True)


@pytest.mark.gpu
@pytest.mark.parametrize("at", ["end", "start"])
def test_cache_reads_stay_inside(at):
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs a CUDA device")
    r = subprocess.run([sys.executable, os.path.abspath(__file__), at], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("ok ") == len(CASES) + 1 and "control" in r.stdout, r.stdout


if __name__ == "__main__":
    _child(sys.argv[1])
