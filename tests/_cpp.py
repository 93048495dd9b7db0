"""Build recipe for the C++ API test program (tests/cpp/test_cpp_api.cpp)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_cpp_test(out_dir):
    from paper_2501_16383_b200 import build

    import oracle

    build.build()
    oracle.build(ref=False)
    exe = os.path.join(out_dir, "test_cpp_api")
    lib = os.path.join(ROOT, "paper_2501_16383_b200", "_lib")
    orc = os.path.join(ROOT, "oracle", "_build")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "oracle"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), "-o", exe,
           "-L", lib, "-lrotatekv_b200", "-L", orc, "-lrkv_oracle", "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{lib}:{orc}:/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    return exe
