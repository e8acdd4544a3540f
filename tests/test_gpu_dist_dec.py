"""The eigen-decoupled slab-sharded solve (dist.DecoupledSharded)
on one GPU: every slab's plans, pack/unpack and all-to-all data movement run
in one process (dist.decoupled_emulated_solve), against the reference solver
on identical seeded inputs, for 1-8 slabs; and the single-rank path through
torch.distributed (world size 1, NCCL)."""
import os

import numpy as np
import pytest

from conftest import rel_diff

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,dims,nslabs", [
    (2, (24, 20, 18), 1), (2, (24, 20, 18), 2), (2, (33, 20, 27), 3), (1, (32, 32, 32), 4),
    (2, (64, 48, 40), 8), (2, (20, 12, 10, 16), 3), (2, (40, 30, 64), 5)])
def test_decoupled_sharded_emulated(ref, gpu, kind, dims, nslabs):
    from paper_1905_09539_b200.dist import decoupled_emulated_solve
    from paper_1905_09539_b200.plan import Context
    p = gpu.make_problem(kind, dims, seed=21)
    fs = [gpu.schur(a) for a in p.coeffs]
    ctx = Context(0)
    x = decoupled_emulated_solve(ctx, [f[1] for f in fs], [f[0] for f in fs], p.rhs, nslabs)
    want, info = ref.solve_laplace(p.coeffs, p.rhs, strategy=0, arithmetic=1)
    err = rel_diff(x, want)
    res = ref.residual_laplace(p.coeffs, p.rhs, x)
    print(f"{dims} x {nslabs} slabs: rel={err:.2e} res={res:.2e}")
    assert err <= 1e-10, err
    assert res <= 1e-12, res


@pytest.mark.parametrize("kind,dims,nslabs,chunks", [(2, (24, 20, 18), 2, 2), (2, (33, 20, 27), 3, 4),
                                                     (2, (20, 12, 10, 16), 3, 3)])
def test_decoupled_sharded_emulated_chunk_plans(ref, gpu, kind, dims, nslabs, chunks):
    """Phase A on the per-chunk plans of the pipelined solve (ragged chunks,
    snapped off the 2x2 cells of the last mode)."""
    from paper_1905_09539_b200.dist import decoupled_emulated_solve
    from paper_1905_09539_b200.plan import Context
    p = gpu.make_problem(kind, dims, seed=23)
    fs = [gpu.schur(a) for a in p.coeffs]
    x = decoupled_emulated_solve(Context(0), [f[1] for f in fs], [f[0] for f in fs], p.rhs, nslabs, chunks=chunks)
    want, _ = ref.solve_laplace(p.coeffs, p.rhs, strategy=0, arithmetic=1)
    assert rel_diff(x, want) <= 1e-10
    assert ref.residual_laplace(p.coeffs, p.rhs, x) <= 1e-12


@pytest.mark.parametrize("chunks,dims", [(1, (64, 64, 64)), (3, (64, 64, 64)), (4, (40, 24, 50))])
def test_decoupled_sharded_world1_nccl(ref, gpu, chunks, dims):
    """The real orchestration (NCCL process group of one rank); chunks > 1:
    the pipelined exchanges (list all_to_all on the communication stream,
    event-ordered against the compute stream)."""
    import torch
    import torch.distributed as dist
    from paper_1905_09539_b200.dist import DecoupledSharded, DeviceDecoupled
    from paper_1905_09539_b200.plan import Context
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(29561 + chunks)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        p = gpu.make_problem(1 if dims[0] == 64 else 2, dims, seed=22)
        fs = [gpu.schur(a) for a in p.coeffs]
        ctx = Context(0)
        be = DeviceDecoupled(ctx, 0, 1, [f[1] for f in fs], [f[0] for f in fs], chunks=chunks)
        assert len(be.cb) == chunks + 1
        sh = DecoupledSharded(be)
        b = torch.from_numpy(np.ascontiguousarray(p.rhs).reshape(-1, order="F")).cuda()
        x = torch.empty_like(b)
        torch.cuda.synchronize()
        for _ in range(3):  # repeated solves reuse every buffer and flag
            sh.solve(b, x, check=True)
        torch.cuda.synchronize()
        xs = x.cpu().numpy().reshape(p.rhs.shape, order="F")
        want, _ = ref.solve_laplace(p.coeffs, p.rhs, strategy=0, arithmetic=1)
        assert rel_diff(xs, want) <= 1e-10
        be.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows,n0,b0", [(7, 24, [0, 24]), (5, 24, [0, 10, 24]), (33, 70, [0, 9, 9, 40, 70]),
                                        (4, 1024, [0, 130, 256, 700, 1024]), (1000, 12, [0, 5, 12])])
def test_slab_pack_kernel(gpu, rows, n0, b0):
    """tsg_slab_pack (the all-to-all send layout) against numpy, both directions;
    ragged and empty segments, n0 below a warp and above a block."""
    import ctypes

    import torch
    from paper_1905_09539_b200._lib import lib
    from paper_1905_09539_b200.plan import Context
    ctx = Context(0)
    P = len(b0) - 1
    rng = np.random.default_rng(rows * n0)
    v = rng.standard_normal((rows, n0))
    want = np.concatenate([v[:, b0[q]:b0[q + 1]].reshape(-1) for q in range(P)])
    src = torch.from_numpy(v.reshape(-1)).cuda()
    dst = torch.zeros_like(src)
    bb = (ctypes.c_int * (P + 1))(*b0)
    for direction, a, b in ((0, src, dst), (1, dst, torch.zeros_like(src))):
        rc = lib().tsg_slab_pack(ctx.h, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), rows, n0, P,
                                 bb, direction, ctypes.c_void_p(ctx.stream_ptr()))
        assert rc == 0, ctx.last_error()
        torch.cuda.synchronize()
        got = b.cpu().numpy()
        assert np.array_equal(got, want if direction == 0 else v.reshape(-1))
    bad = (ctypes.c_int * (P + 1))(*([1] + list(b0[1:])))
    assert lib().tsg_slab_pack(ctx.h, ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), rows, n0, P,
                               bad, 0, None) != 0
