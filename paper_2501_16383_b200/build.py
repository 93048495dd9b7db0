"""Build the in-tree sm_100a library (plain nvcc, no torch extension).

    python -m paper_2501_16383_b200.build

produces paper_2501_16383_b200/_lib/librotatekv_b200.so, a C-ABI shared
library (include/rotatekv/rotatekv.h) that the Python host layer loads with
ctypes and that a C/C++ caller links directly.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "librotatekv_b200.so")
INCLUDE = os.path.join(ROOT, "include")
SOURCES = ["rkv_api.cu", "rkv_runtime.cu", "rkv_plan.cu", "quantize_kv.cu", "generic.cu", "decode_attention.cu", "decode_mma.cu", "prefill.cu", "sink_detect.cu"]
HEADERS = ["rkv_common.cuh", "rkv_internal.h", "rkv_layout.h", "rkv_mma.cuh", "rkv_umma.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
              "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every source to an object (in parallel; an object is rebuilt when
    its source, a shared header or the compiler flags changed) and link the
    shared library."""
    from concurrent.futures import ThreadPoolExecutor

    hdrs = [os.path.join(CSRC, f) for f in HEADERS] + [os.path.join(INCLUDE, "rotatekv", "rotatekv.h")]
    extra = os.environ.get("RKV_NVCC_EXTRA", "").split()  # experiment flags (e.g. -DRKV_DEC_TRACE)
    os.makedirs(LIBDIR, exist_ok=True)
    stamp = os.path.join(LIBDIR, ".flags")
    flags = " ".join(ARCH + NVCC_FLAGS + extra)
    flags_changed = not os.path.exists(stamp) or open(stamp).read() != flags
    objs, jobs = [], []
    for src in SOURCES:
        obj = os.path.join(LIBDIR, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or flags_changed or _stale(obj, [os.path.join(CSRC, src)] + hdrs):
            cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, *extra, "-I", INCLUDE, "-c", os.path.join(CSRC, src), "-o", obj]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)
    if not jobs and not _stale(LIB, objs):
        build_e2e_cpp()
        return LIB

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    with open(stamp, "w") as f:
        f.write(flags)
    tmp = LIB + ".tmp"
    subprocess.run([_nvcc(), *ARCH, "-shared", "-o", tmp, *objs], check=True)
    os.replace(tmp, LIB)
    build_e2e_cpp(force=True)
    return LIB


E2E_CPP = os.path.join(LIBDIR, "rkv_e2e_cpp")


def build_e2e_cpp(force: bool = False) -> str:
    """The C++-API decode-step program bench.py times for `e2e_cpp`
    (csrc/e2e_cpp.cu, linked against the library with an $ORIGIN rpath)."""
    src = os.path.join(CSRC, "e2e_cpp.cu")
    hpp = os.path.join(INCLUDE, "rotatekv", "rotatekv.hpp")
    if not force and not _stale(E2E_CPP, [src, hpp, LIB]):
        return E2E_CPP
    subprocess.run([_nvcc(), *ARCH, "-O2", "-std=c++17", "-I", INCLUDE, src, "-o", E2E_CPP + ".tmp", "-L", LIBDIR,
                    "-lrotatekv_b200", "-Xlinker", "-rpath,$ORIGIN"], check=True)
    os.replace(E2E_CPP + ".tmp", E2E_CPP)
    return E2E_CPP


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
