"""World-size-2 (and 3) CPU runs of the sharded-solve orchestration
(paper_1905_09539_b200.dist.ShardedLaplace) over torch.distributed gloo.

The device steps are replaced by ``CpuSlabs``, a numpy stand-in that follows
the tsg_dplan step semantics of include/tsylv_gpu.h (padded send slots of
rmax rows, gather of nranks slots, last-mode transforms against the
zero-padded rows of U^T / U); its reduced solve gathers the transformed slabs
and runs the oracle recursion (test infrastructure).  The slab bounds come
from the library's host function tsg_slab_bounds (no GPU needed).  The CUDA
implementation of the same steps is checked on the GPU in emulated mode
(tests/test_gpu_dist.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restate as R


class CpuSlabs:
    def __init__(self, rank, nranks, T, U):
        from paper_1905_09539_b200.dist import slab_bounds
        self.rank, self.nranks, self.emulate = rank, nranks, False
        self.T, self.U = T, U
        self.dims = [t.shape[0] for t in T]
        self.bounds = slab_bounds(self.dims[-1], T[-1], nranks)
        self.rows = [b1 - b0 for b0, b1 in zip(self.bounds, self.bounds[1:])]
        self.rmax = max(self.rows)
        self.plane = int(np.prod(self.dims[:-1]))
        self.send = torch.zeros(self.rmax * self.plane, dtype=torch.float64)
        self.gather = torch.zeros(nranks * self.rmax * self.plane, dtype=torch.float64)
        self.xt = None

    def _pad(self, mat_rows_of):
        """rows R_r of a matrix, columns scattered to the padded gather layout"""
        lo, r, K = self.bounds[self.rank], self.rows[self.rank], self.nranks * self.rmax
        out = np.zeros((r, K))
        for q in range(self.nranks):
            q0 = self.bounds[q]
            out[:, q * self.rmax:q * self.rmax + self.rows[q]] = mat_rows_of[lo:lo + r, q0:q0 + self.rows[q]]
        return out

    def _slab_shape(self, q):
        return tuple(self.dims[:-1]) + (self.rows[q],)

    def _to_send(self, y):
        self.send.zero_()
        self.send[:y.size] = torch.from_numpy(y.ravel(order="F"))

    def forward_local(self, b, stream):
        y = b.numpy().reshape(self._slab_shape(self.rank), order="F")
        for m in range(len(self.dims) - 1):
            y = R.mode_multiply(y, self.U[m].T, m)
        self._to_send(y)

    def _gathered(self):
        shp = tuple(self.dims[:-1]) + (self.nranks * self.rmax,)
        return self.gather.numpy().reshape(shp, order="F")

    def forward_split(self, stream):
        d = len(self.dims)
        self.xt = R.mode_multiply(self._gathered(), self._pad(self.U[-1].T), d - 1)

    def solve(self, stream, group=None):
        # gather B~ (padded slabs), solve the whole reduced problem, keep ours
        d = len(self.dims)
        mine = torch.zeros(self.rmax * self.plane, dtype=torch.float64)
        mine[:self.xt.size] = torch.from_numpy(self.xt.ravel(order="F"))
        allb = torch.zeros(self.nranks * self.rmax * self.plane, dtype=torch.float64)
        dist.all_gather_into_tensor(allb, mine, group=group)
        parts = []
        for q in range(self.nranks):
            seg = allb[q * self.rmax * self.plane:(q * self.rmax + self.rows[q]) * self.plane]
            parts.append(seg.numpy().reshape(self._slab_shape(q), order="F"))
        bt = np.concatenate(parts, axis=d - 1)
        xt = R.laplace_recursive(self.T, bt, 4)
        lo = self.bounds[self.rank]
        self.xt = np.asfortranarray(xt[..., lo:lo + self.rows[self.rank]])

    def back_local(self, stream):
        y = self.xt
        for m in range(len(self.dims) - 1):
            y = R.mode_multiply(y, self.U[m], m)
        self._to_send(y)

    def back_split(self, x, stream):
        d = len(self.dims)
        y = R.mode_multiply(self._gathered(), self._pad(self.U[-1]), d - 1)
        x.copy_(torch.from_numpy(y.ravel(order="F")))

    def status(self, stream):
        pass


def _worker(rank, world, port, dims, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1905_09539_b200.dist import ShardedLaplace
        coeffs, _, rhs = R.baseline_problem(2, dims, seed=7)
        f = [R.schur(a) for a in coeffs]   # (U, T) per mode, shared setup
        U = [u for u, _ in f]
        T = [t for _, t in f]
        be = CpuSlabs(rank, world, T, U)
        lo, hi = be.bounds[rank], be.bounds[rank + 1]
        b = torch.from_numpy(np.asfortranarray(rhs[..., lo:hi]).ravel(order="F").copy())
        x = torch.zeros_like(b)
        ShardedLaplace(be).solve(b, x)
        want = R.solve_laplace(coeffs, rhs, n_min=4)[..., lo:hi]
        got = x.numpy().reshape(want.shape, order="F")
        err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
        q.put((rank, lo, hi, err))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,dims", [(2, (6, 5, 24)), (3, (5, 4, 27))])
def test_sharded_orchestration_gloo(world, dims):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == 0 and res[-1][2] == dims[-1]
    for (r0, lo0, hi0, _), (r1, lo1, hi1, _) in zip(res, res[1:]):
        assert hi0 == lo1  # slabs tile the last mode
    for r, lo, hi, err in res:
        assert hi > lo
        assert err < 1e-12, (r, err)


def test_slab_bounds_tile_aligned_and_balanced():
    from paper_1905_09539_b200.dist import slab_bounds
    coeffs, _, _ = R.baseline_problem(2, (256,), seed=1)
    _, t = R.schur(coeffs[0])
    for k in (1, 2, 3, 4, 8):
        b = slab_bounds(256, t, k)
        assert b[0] == 0 and b[-1] == 256 and len(b) == k + 1
        rows = np.diff(b)
        assert rows.min() > 0 and rows.max() - rows.min() <= 16
        for x in b[1:-1]:
            assert t[x, x - 1] == 0.0  # never inside a 2x2 Schur block
    with pytest.raises(ValueError):
        slab_bounds(16, t[:16, :16], 4)  # fewer tiles than ranks
