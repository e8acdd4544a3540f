"""Race screen (compute-sanitizer is closed on this GPU pool):
every kernel family solves the same problem repeatedly and must return
bit-identical results.  The kernels hand data between warps and CTAs through
shared-memory barriers, ld.acquire / st.release flags, mbarrier rings and
dataflow counters; none of them accumulates in a schedule-dependent order, so
any run-to-run difference is a missed synchronisation.  Each result is also
checked against the reference solver."""
import os

import numpy as np
import pytest

from conftest import rel_diff

pytestmark = pytest.mark.gpu

REPEATS = 12

# (name, kind, dims, plan knobs) — the families of tools/sanitize_cases.py
CASES = [
    ("tile-DAG 8^3 (lap3)", 1, (24, 20, 16), {"TSG_DECOUPLE": "0"}),
    ("tile-DAG 16^3 TMA ring (lap16)", 2, (36, 34, 33), {"TSG_LAP16": "1", "TSG_DECOUPLE": "0"}),
    ("tile-DAG order 6 (lapd)", 2, (5, 4, 4, 3, 3, 3), {"TSG_DECOUPLE": "0"}),
    ("decoupled, register kernel", 2, (12, 10, 8), {}),
    ("decoupled, register kernel, order 6", 2, (7, 6, 9, 5, 4, 6), {}),
    ("decoupled, team kernel", 2, (16, 40, 33), {}),
    ("decoupled, team kernel, long fibres + TMA GEMM", 2, (72, 130, 65), {}),
    ("fused small-mode passes", 2, (24, 24, 16, 16), {}),
    ("gsylv tile-DAG (gsyd)", 5, (20, 4, 4, 4), {"TSG_DECOUPLE": "0"}),
    ("gsylv decoupled pencil fibres", 5, (40, 8, 8, 8), {}),
]


@pytest.mark.parametrize("name,kind,dims,env", CASES, ids=[c[0] for c in CASES])
def test_repeated_solves_bit_identical(ref, gpu, name, kind, dims, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        cfg = gpu.SolverConfig(strategy=gpu.Strategy.recursion_only,
                               arithmetic=gpu.Arithmetic.real_quasitriangular)
        p = gpu.make_problem(kind, dims, seed=31)
        solve = gpu.solve_gsylv if kind == 5 else gpu.solve_laplace
        first = np.array(solve(p, cfg).solution, copy=True)
        for k in range(1, REPEATS):
            again = solve(p, cfg).solution
            assert np.array_equal(first, again), f"{name}: solve {k} differs from solve 0 " \
                f"(max |diff| {np.abs(first - again).max():.3e})"
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    if kind == 5:
        want, _ = ref.solve_gsylv(p.coeffs, p.c, p.rhs, strategy=0, arithmetic=1)
    else:
        want, _ = ref.solve_laplace(p.coeffs, p.rhs, strategy=0, arithmetic=1)
    assert rel_diff(first, want) <= 1e-10


def test_repeated_complex_solves_bit_identical(gpu):
    for fam, dims in (("laplace", (20, 70, 12)), ("gsylv", (70, 6, 5))):
        p = gpu.random_problem(fam, dims, seed=5)
        solve = gpu.solve_laplace if fam == "laplace" else gpu.solve_gsylv
        first = np.array(solve(p).solution, copy=True)
        for k in range(1, 6):
            assert np.array_equal(first, solve(p).solution), (fam, k)
