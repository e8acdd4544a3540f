"""C++ users of the drop-in headers: builds tests/cpp/*.cpp against
include/ and libtsylv_gpu.so (g++, the same OpenBLAS the library links for
the Schur setup) and runs them (the bench harness, include/tsylv/bench.hpp,
checked the way the reference's tests/test_bench.cpp checks its own)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(src, out):
    from paper_1905_09539_b200 import build as b
    bdir, blib = b.blas_lib()
    libdir = os.path.join(ROOT, "paper_1905_09539_b200")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(b.cuda_home(), "include"),
           src, "-o", out, os.path.join(libdir, "libtsylv_gpu.so"), blib,
           f"-Wl,--disable-new-dtags,-rpath,{libdir}:{bdir}", "-lpthread"]
    subprocess.run(cmd, check=True)


def test_bench_harness_cpp(tmp_path):
    exe = str(tmp_path / "test_bench_dropin")
    _build(os.path.join(ROOT, "tests", "cpp", "test_bench_dropin.cpp"), exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    print(r.stderr)
    assert r.returncode == 0, r.stderr
    assert "PASS" in r.stdout
