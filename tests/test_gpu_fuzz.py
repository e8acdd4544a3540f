"""Seeded shape fuzz of the full pipeline (forward transforms, dataflow solve,
back transforms, and every overlap: back-transform gate, slab chain,
trailing cube) against the reference build on identical inputs.  Shapes are
drawn so that each kernel family is hit: 8^3 tiles (lap3), 16^3 TMA tiles
with and without the trailing cube (lap16), order 4..6 (lapd), gsylv
(gsyd), small-mode transform pairs (16/24/32/40 extents), odd extents
(2x2 Schur blocks on tile boundaries)."""
import numpy as np
import pytest

from conftest import rel_diff

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

REL = 1e-10
RES = 1e-12


def _shapes():
    # TSG_FUZZ_SEEDS=k runs k seeded draws (default one)
    import os
    out = []
    for seed in range(2026, 2026 + int(os.environ.get("TSG_FUZZ_SEEDS", "1"))):
        out += _draw(np.random.default_rng(seed))
    return out


def _draw(rng):
    out = []
    for _ in range(4):  # lap3 / generic order 3
        out.append((2, tuple(int(v) for v in rng.integers(20, 90, 3)), {}))
    for _ in range(3):  # 16^3 tiles forced, some with a cube
        out.append((2, tuple(int(v) for v in rng.integers(100, 180, 3)), {"TSG_LAP16": "1", "TSG_CUBE": "2",
                                                                          "TSG_CUBE_GRID": "4"}))
    for d in (4, 5, 6):  # lapd
        out.append((2, tuple(int(v) for v in rng.integers(5, 13, d)), {}))
    out.append((2, (24, 40, 16, 11), {}))  # small-mode pairs
    out.append((5, (37, 9, 9, 9), {}))     # gsylv
    out.append((5, (50, 24, 24), {}))
    # small extents (fused transform passes) mixed with odd ones, any position
    small = [16, 24, 32, 40]
    for _ in range(10):
        d = int(rng.integers(2, 5))
        dims = [int(rng.choice(small)) if rng.random() < 0.5 else int(rng.integers(3, 30)) for _ in range(d)]
        if int(np.prod(dims)) > 400_000:
            dims[-1] = 3
        out.append((2, tuple(dims), {}))
    for _ in range(3):
        n0 = int(rng.integers(5, 40))
        nt = int(rng.choice(small + [7, 9]))
        out.append((5, (n0, nt, nt), {}))
    return out


@pytest.mark.parametrize("kind,dims,env", _shapes())
def test_fuzz_pipeline(gpu, ref, kind, dims, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    p = gpu.make_problem(kind, dims, seed=sum(dims))
    cfg = gpu.SolverConfig(strategy=gpu.Strategy.recursion_only, arithmetic=gpu.Arithmetic.real_quasitriangular)
    if kind == 5:
        want, _ = ref.solve_gsylv(p.coeffs, p.c, p.rhs, strategy=0, arithmetic=1)
        rep = gpu.solve_gsylv(p, cfg)
    else:
        want, _ = ref.solve_laplace(p.coeffs, p.rhs, strategy=0, arithmetic=1)
        rep = gpu.solve_laplace(p, cfg)
    assert rel_diff(rep.solution, want) < REL
    assert rep.residual < RES
