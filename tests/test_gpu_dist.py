"""Slab-sharded solve on one GPU in emulated mode: one
process owns every slab (separate device buffers), the transforms run per
slab against the zero-padded gather layout and one dataflow kernel reads the
slabs through the same per-slab addressing the multi-GPU path uses for peer
mappings.  Checked against the reference CPU solver (oracle/_ref)."""
import numpy as np
import pytest

from conftest import rel_diff

pytestmark = pytest.mark.gpu


def _solve_emulated(gpu, coeffs, rhs, nranks):
    import torch
    from paper_1905_09539_b200.dist import DeviceSlabs, ShardedLaplace
    from paper_1905_09539_b200.plan import Context
    f = [gpu.schur(a) for a in coeffs]
    ctx = Context(0)
    be = DeviceSlabs(ctx, 0, nranks, [t for _, t in f], [u for u, _ in f], emulate=True)
    sl = ShardedLaplace(be)
    b = torch.from_numpy(np.asfortranarray(rhs).ravel(order="F").copy()).cuda()
    x = torch.empty_like(b)
    stream = torch.cuda.current_stream().cuda_stream
    sl.solve(b, x, stream=stream, check=True)
    torch.cuda.synchronize()
    out = x.cpu().numpy().reshape(rhs.shape, order="F")
    return out, be.bounds


@pytest.mark.parametrize("nranks", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("dims", [(40, 36, 72), (64, 64, 64)])
def test_sharded_emulated_matches_reference(gpu, ref, dims, nranks):
    p = gpu.make_problem(2, dims, seed=3)
    want, _ = ref.solve_laplace(p.coeffs, p.rhs, strategy=0, arithmetic=1)
    got, bounds = _solve_emulated(gpu, p.coeffs, p.rhs, nranks)
    assert len(bounds) == nranks + 1 and bounds[0] == 0 and bounds[-1] == dims[-1]
    assert all(b1 > b0 for b0, b1 in zip(bounds, bounds[1:]))
    assert rel_diff(got, want) < 1e-10
    assert ref.residual_laplace(p.coeffs, p.rhs, got) < 1e-12


def test_sharded_emulated_convection_diffusion(gpu, ref):
    p = gpu.make_problem(1, (32, 24, 40), seed=1)
    want, _ = ref.solve_laplace(p.coeffs, p.rhs, strategy=0, arithmetic=1)
    got, _ = _solve_emulated(gpu, p.coeffs, p.rhs, 4)
    assert rel_diff(got, want) < 1e-10


def test_sharded_emulated_repeated_epochs(gpu, ref):
    """Flags are epoch-stamped, never reset: solves back to back must agree."""
    import torch
    from paper_1905_09539_b200.dist import DeviceSlabs, ShardedLaplace
    from paper_1905_09539_b200.plan import Context
    p = gpu.make_problem(2, (24, 20, 33), seed=4)
    f = [gpu.schur(a) for a in p.coeffs]
    be = DeviceSlabs(Context(0), 0, 3, [t for _, t in f], [u for u, _ in f], emulate=True)
    sl = ShardedLaplace(be)
    want, _ = ref.solve_laplace(p.coeffs, p.rhs, strategy=0, arithmetic=1)
    b = torch.from_numpy(p.rhs.ravel(order="F").copy()).cuda()
    for _ in range(4):
        x = torch.zeros_like(b)
        sl.solve(b, x, stream=torch.cuda.current_stream().cuda_stream, check=True)
        got = x.cpu().numpy().reshape(p.rhs.shape, order="F")
        assert rel_diff(got, want) < 1e-10
