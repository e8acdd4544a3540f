"""Eigen-decoupled fibre solve (solve_fibre.cu) against the
reference solver on identical seeded inputs, and against the tile-DAG
kernels (TSG_DECOUPLE=0) on the same plan inputs.

Shapes cover: the order-3 convection-diffusion family (C1), the
G/sqrt(n)+3I family (C2-C4) at small sizes, order 4-6 (C3-type), order 2,
odd extents, free modes of both parities and 1x1/2x2 cell mixes."""
import os

import numpy as np
import pytest

from conftest import rel_diff

pytestmark = pytest.mark.gpu

SHAPES = [
    (1, (32, 32, 32)), (1, (20, 24, 16)), (2, (12, 10, 8)), (2, (40, 33, 17)), (2, (64, 64, 64)),
    (2, (9, 48)), (2, (24, 24, 24, 24)), (2, (7, 6, 5, 4)), (2, (5, 4, 4, 3, 3, 3)),
    (2, (24, 24, 6, 5, 4)), (2, (3, 3, 3, 3, 3, 3)), (2, (31, 5, 29)),
]


def _plan(gpu, p, **kw):
    from paper_1905_09539_b200.plan import Context, Plan
    ctx = Context(0)
    fs = [gpu.schur(a) for a in p.coeffs]
    return ctx, Plan(ctx, 0, [f[1] for f in fs], [f[0] for f in fs], **kw)


def _solve(plan, p):
    b = np.asfortranarray(p.rhs)
    x = np.zeros_like(b)
    plan.execute_host(b, x)
    return x


@pytest.mark.parametrize("kind,dims", SHAPES)
def test_decoupled_vs_reference(ref, gpu, kind, dims):
    p = gpu.make_problem(kind, dims, seed=11)
    ctx, plan = _plan(gpu, p)
    desc = plan.describe()
    assert desc.startswith("decoupled"), desc
    x = _solve(plan, p)
    want, info = ref.solve_laplace(p.coeffs, p.rhs, strategy=0, arithmetic=1)
    err = rel_diff(x, want)
    res = ref.residual_laplace(p.coeffs, p.rhs, x)
    print(f"{dims}: {desc} rel={err:.2e} res={res:.2e}")
    assert err <= 1e-10, err
    assert res <= 1e-12, res
    plan.close()


@pytest.mark.parametrize("kind,dims", [(2, (24, 24, 24, 24)), (1, (32, 32, 32)), (2, (7, 6, 5, 4))])
def test_decoupled_matches_tile_kernels(gpu, kind, dims):
    p = gpu.make_problem(kind, dims, seed=12)
    ctx, plan = _plan(gpu, p)
    assert plan.describe().startswith("decoupled")
    x1 = _solve(plan, p)
    plan.close()
    os.environ["TSG_DECOUPLE"] = "0"
    try:
        ctx2, plan2 = _plan(gpu, p)
        assert not plan2.describe().startswith("decoupled")
        x2 = _solve(plan2, p)
        plan2.close()
    finally:
        del os.environ["TSG_DECOUPLE"]
    assert rel_diff(x1, x2) <= 1e-11


def test_decoupled_rejects_ill_conditioned_bases(gpu):
    """A mode whose eigenbasis is far from orthogonal (a nearly defective
    Jordan-like block) is not decoupled: the plan keeps the tile kernels."""
    n = 16
    a = 2.0 * np.eye(n) + np.diag(np.full(n - 1, 1.0), 1) + np.diag(np.linspace(0, 1e-6, n))
    p = gpu.LaplaceProblem([a, a.copy(), a.copy()], np.ones((n, n, n), order="F"))
    ctx, plan = _plan(gpu, p)
    assert not plan.describe().startswith("decoupled"), plan.describe()
    plan.close()


def test_decoupled_singular_operator(gpu):
    """lambda(A0) + lambda(A1) + lambda(A2) = 0 for one tuple: the fibre
    solve reports the zero pivot (singular_error through the drop-in)."""
    a0 = np.diag([1.0, 2.0, 3.0, 4.0])
    a1 = np.diag([0.5, -3.0, 1.0, 2.0])
    a2 = np.diag([1.0, 1.5, 2.5, 3.5])  # 2 + (-3) + 1 = 0
    p = gpu.LaplaceProblem([a0, a1, a2], np.ones((4, 4, 4), order="F"))
    ctx, plan = _plan(gpu, p)
    b = np.asfortranarray(p.rhs)
    x = np.zeros_like(b)
    with pytest.raises(gpu.gpu_error):
        rep = plan.execute_host(b, x)
        if rep.zero_pivot_index >= 0:
            raise gpu.gpu_error("singular")
    plan.close()


# ---- gsylv: A X + B X (C (x) ... (x) C) = D with the tail modes decoupled ----
GS_SHAPES = [(5, (32, 6, 6, 6)), (5, (48, 8, 8)), (5, (40, 10)), (5, (33, 7, 7, 7)), (5, (64, 12, 12, 12)),
             (5, (29, 3, 3, 3, 3))]


def _gs_plan(gpu, p):
    from paper_1905_09539_b200.plan import Context, Plan
    ctx = Context(0)
    q, z, s, tc = gpu.qz(p.coeffs[0], p.c)
    fs = [gpu.schur(a) for a in p.coeffs[1:]]
    return ctx, Plan(ctx, 1, [s] + [f[1] for f in fs], [q] + [f[0] for f in fs], Tc=tc, Z=z)


@pytest.mark.parametrize("kind,dims", GS_SHAPES)
def test_decoupled_gsylv_vs_reference(ref, gpu, kind, dims):
    """The pencil fibre solve (S + z Tc) x = b, z the product of the tail
    eigenvalues, against the reference solve_gsylv (gsylv.hpp:311-331)."""
    p = gpu.make_problem(kind, dims, seed=13)
    ctx, plan = _gs_plan(gpu, p)
    desc = plan.describe()
    assert desc.startswith("decoupled"), desc
    x = _solve(plan, p)
    want, info = ref.solve_gsylv(p.coeffs, p.c, p.rhs, strategy=0, arithmetic=1)
    err = rel_diff(x, want)
    res = ref.residual_gsylv(p.coeffs, p.c, p.rhs, x)
    print(f"gsylv {dims}: {desc} rel={err:.2e} res={res:.2e}")
    assert err <= 1e-10, err
    assert res <= 1e-12, res
    plan.close()


def test_decoupled_gsylv_matches_tile_kernels(gpu):
    p = gpu.make_problem(5, (40, 8, 8, 8), seed=14)
    ctx, plan = _gs_plan(gpu, p)
    assert plan.describe().startswith("decoupled")
    x1 = _solve(plan, p)
    plan.close()
    os.environ["TSG_DECOUPLE"] = "0"
    try:
        ctx2, plan2 = _gs_plan(gpu, p)
        assert not plan2.describe().startswith("decoupled")
        x2 = _solve(plan2, p)
        plan2.close()
    finally:
        del os.environ["TSG_DECOUPLE"]
    assert rel_diff(x1, x2) <= 1e-11
