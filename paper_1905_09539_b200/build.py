"""In-tree build of the sm_100a library ``libtsylv_gpu.so``.

Compiles the hand-written CUDA kernels (csrc/*.cu) for
``-gencode arch=compute_100a,code=sm_100a`` with ``-lineinfo`` and the C++
host side (C-ABI plans + the header-only drop-in facade, csrc/*.cpp), and
links them against the LAPACK-exporting OpenBLAS that also backs the oracle
(shared Schur/QZ setup).  The .so is written next to this file so
it travels to the GPU box with the repo snapshot.

    python -m paper_1905_09539_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import site
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libtsylv_gpu.so")
CLI = os.path.join(HERE, "bin", "tsylv")
CLI_SRC = os.path.join(ROOT, "tools", "tsylv_cli.cpp")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def cuda_home() -> str:
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return os.path.dirname(os.path.dirname(os.path.realpath(nvcc)))


def blas_lib() -> tuple[str, str]:
    """LP64 OpenBLAS exporting dgees_/dgges_ (opencv wheel copy)."""
    cands = []
    for p in site.getsitepackages() + [site.getusersitepackages()]:
        cands += glob.glob(os.path.join(p, "opencv_python_headless.libs", "libopenblasp-*.so"))
    if not cands:
        raise RuntimeError("no LAPACK-exporting OpenBLAS found (opencv_python_headless.libs)")
    lib = cands[0]
    return os.path.dirname(lib), lib


def json_include() -> str | None:
    """Directory holding nlohmann/json.hpp (the copy cudnn_frontend ships in
    this image), for the JSON problem files (include/tsylv/io.hpp)."""
    for p in site.getsitepackages() + [site.getusersitepackages()]:
        for hit in glob.glob(os.path.join(p, "include", "*", "thirdparty", "nlohmann", "json.hpp")):
            return os.path.dirname(os.path.dirname(hit))
    return None


def cxx_user_cmd(src: str, out: str, opt: str = "-O2") -> list[str]:
    """g++ command for a C++ user of the drop-in headers: include/, the
    library, its OpenBLAS and (when present) nlohmann/json."""
    bdir, blib = blas_lib()
    jinc = json_include()
    cmd = ["g++", "-std=c++20", opt, "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda_home(), "include")]
    if jinc:
        cmd += ["-I", jinc]
    return cmd + [src, "-o", out, LIB, blib, f"-Wl,--disable-new-dtags,-rpath,{HERE}:{bdir}", "-lpthread"]


def build_cli(force: bool = False, verbose: bool = False) -> str | None:
    """The command-line front end (tools/tsylv_cli.cpp, the reference's
    tools/tsylv.cpp) as paper_1905_09539_b200/bin/tsylv; None without
    nlohmann/json."""
    if json_include() is None:
        return None
    headers = glob.glob(os.path.join(ROOT, "include", "tsylv", "*.hpp")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    if force or _newer(CLI, [CLI_SRC, LIB] + headers):
        os.makedirs(os.path.dirname(CLI), exist_ok=True)
        _run(cxx_user_cmd(CLI_SRC, CLI), verbose)
    return CLI


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    headers += glob.glob(os.path.join(ROOT, "include", "*.h"))
    headers += glob.glob(os.path.join(ROOT, "include", "tsylv", "*.hpp"))
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    cuda_inc = ["-I", os.path.join(cuda_home(), "include")]
    jobs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        extra = os.environ.get("TSG_NVCC_FLAGS", "").split()
        cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-diag-suppress", "177", *extra, *inc, "-c", src, "-o", obj]
        jobs.append((obj, [src] + headers, cmd))
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cpp"))):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        # macro definitions of TSG_NVCC_FLAGS apply to the host side too
        # (e.g. -DTSG_DEVTOOLS: the development probes, tools/README.md)
        defs = [f for f in os.environ.get("TSG_NVCC_FLAGS", "").split() if f.startswith("-D")]
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-Wno-unused-function", *defs,
               *inc, *cuda_inc, "-c", src, "-o", obj]
        jobs.append((obj, [src] + headers, cmd))
    todo = [(o, c) for o, deps, c in jobs if force or _newer(o, deps)]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(lambda oc: _run(oc[1], verbose), todo))
    objs = [o for o, _, _ in jobs]
    if force or todo or _newer(LIB, objs):
        bdir, blib = blas_lib()
        _run(["nvcc", *ARCH, "-shared", "-o", LIB, *objs, blib,
              "-Xlinker", f"--disable-new-dtags,-rpath,{bdir}", "-lpthread"], verbose)
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
    print(build_cli(a.force, a.verbose))


if __name__ == "__main__":
    main()
