"""Full BASELINE.json sizes (C1-C5) on the GPU through size-independent
properties: the reference residual gate (<= 1e-12, oracle.hpp:233-268,
computed on the device by tsg_residual) and linearity of the solve
(X(B1 + 2 B2) = X(B1) + 2 X(B2)), with the factors set up once per plan.
The element-wise comparison with the reference solver is done at reduced
sizes in test_gpu_parity.py (the CPU reference needs minutes at C3-C5)."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CONFIGS = {
    "C1": (1, (64, 64, 64)),
    "C2": (2, (256, 256, 256)),
    "C3": (2, (24,) * 6),
    "C4": (2, (1024, 512, 256)),
    "C5": (5, (200, 40, 40, 40)),
}


def _plan(gpu, kind, p):
    from paper_1905_09539_b200.plan import Context, Plan
    ctx = Context(0)
    if kind == 5:
        q, z, s, tc = gpu.qz(p.coeffs[0], p.c)
        fs = [gpu.schur(a) for a in p.coeffs[1:]]
        return ctx, Plan(ctx, 1, [s] + [f[1] for f in fs], [q] + [f[0] for f in fs], Tc=tc, Z=z)
    fs = [gpu.schur(a) for a in p.coeffs]
    return ctx, Plan(ctx, 0, [f[1] for f in fs], [f[0] for f in fs])


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_fullsize_residual_and_linearity(gpu, name):
    kind, dims = CONFIGS[name]
    p = gpu.make_problem(kind, dims, seed=1)
    ctx, plan = _plan(gpu, kind, p)
    b1 = np.asfortranarray(p.rhs)
    rng = np.random.default_rng(7)
    b2 = np.asfortranarray(rng.standard_normal(dims))
    x1 = np.zeros_like(b1)
    x2 = np.zeros_like(b1)
    x3 = np.zeros_like(b1)
    plan.execute_host(b1, x1)
    assert gpu.residual(p, x1) < 1e-12
    plan.execute_host(b2, x2)
    plan.execute_host(np.asfortranarray(b1 + 2.0 * b2), x3)
    lin = np.linalg.norm(x3 - (x1 + 2.0 * x2)) / np.linalg.norm(x3)
    assert lin < 1e-12, lin
