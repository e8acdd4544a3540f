"""World-size-2/3 CPU runs of the eigen-decoupled sharded solve
(paper_1905_09539_b200.dist.DecoupledSharded) over torch.distributed gloo:
the real orchestration (pack, two all_to_all_single exchanges with their
split sizes, unpack) across processes, with a numpy stand-in for the device
phases (test infrastructure, oracle/restate.py):

  phase A/C  mode products with the folded eigenbasis factors
             P_m^-1 U_m^T / U_m P_m (m != f, m < d-1) and U_f^T / U_f,
  phase B    the mode-(d-1) transform and the reduced system on the rank's
             mode-0 slab, solved densely: its mode-0 coefficient is the
             block-diagonal Lambda_0 restricted to the slab (whole cells).

Slab bounds come from the library's host function tsg_slab_bounds (no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restate as R


def _block_eigenbasis(t):
    """Real block-eigenbasis of a quasi-triangular T (the LAPACK dtrevc
    construction): per diagonal cell, the eigenvector by back substitution;
    a complex pair contributes [Re v, Im v] at the cell's two columns."""
    n = t.shape[0]
    p = np.zeros((n, n))
    i = 0
    while i < n:
        s = 2 if i + 1 < n and t[i + 1, i] != 0.0 else 1
        w, v = np.linalg.eig(t[i:i + s, i:i + s])
        lam, vc = w[0], v[:, 0].astype(complex)
        x = np.zeros(n, dtype=complex)
        x[i:i + s] = vc
        if i > 0:
            x[:i] = np.linalg.solve(t[:i, :i] - lam * np.eye(i), -t[:i, i:i + s] @ vc)
        if s == 1:
            p[:, i] = x.real
        else:
            p[:, i], p[:, i + 1] = x.real, x.imag
        i += s
    return p


class CpuDecoupled:
    def __init__(self, rank, nranks, T, U, chunks=1):
        from paper_1905_09539_b200.dist import chunk_bounds, decoupled_free_mode, slab_bounds
        self.rank, self.nranks, self.stream = rank, nranks, 0
        self.T, self.U = T, U
        self.dims = [t.shape[0] for t in T]
        self.f = decoupled_free_mode(self.dims)
        self.bd = slab_bounds(self.dims[-1], T[-1], nranks, tile=1)
        self.b0 = slab_bounds(self.dims[0], T[0], nranks, tile=1)
        # pipeline chunks of every rank's slab (chunks = 1: the slab itself)
        self.cb_all = chunk_bounds(T[-1], self.bd, chunks)
        self.cb = self.cb_all[rank]
        d = len(T)
        self.P = [None if m == self.f else _block_eigenbasis(T[m]) for m in range(d)]
        self.L = [None if m == self.f else np.linalg.solve(self.P[m], T[m] @ self.P[m]) for m in range(d)]

    def empty(self, n):
        return torch.zeros(int(n), dtype=torch.float64)

    def _fwd(self, m):
        return self.U[m].T if m == self.f else np.linalg.solve(self.P[m], self.U[m].T)

    def _bwd(self, m):
        return self.U[m] if m == self.f else self.U[m] @ self.P[m]

    def _shape_a(self, v):
        # a whole slab or one pipeline chunk of it: the extent follows from the length
        return tuple(self.dims[:-1]) + (v.numel() // int(np.prod(self.dims[:-1])),)

    def a_forward(self, b, out):
        y = b.numpy().reshape(self._shape_a(b), order="F")
        for m in range(len(self.dims) - 1):
            y = R.mode_multiply(y, self._fwd(m), m)
        out.copy_(torch.from_numpy(np.asfortranarray(y).reshape(-1, order="F")))

    def a_back(self, x, out):
        y = x.numpy().reshape(self._shape_a(x), order="F")
        for m in range(len(self.dims) - 1):
            y = R.mode_multiply(y, self._bwd(m), m)
        out.copy_(torch.from_numpy(np.asfortranarray(y).reshape(-1, order="F")))

    def b_solve(self, z, out):
        d = len(self.dims)
        q0, q1 = self.b0[self.rank], self.b0[self.rank + 1]
        shp = (q1 - q0,) + tuple(self.dims[1:])
        y = R.mode_multiply(z.numpy().reshape(shp, order="F"), self._fwd(d - 1), d - 1)
        co = [self.L[0][q0:q1, q0:q1]] + [self.T[m] if m == self.f else self.L[m] for m in range(1, d)]
        xs = np.linalg.solve(R.assemble_laplace(co), y.reshape(-1, order="F")).reshape(shp, order="F")
        xs = R.mode_multiply(xs, self._bwd(d - 1), d - 1)
        out.copy_(torch.from_numpy(np.asfortranarray(xs).reshape(-1, order="F")))


def _worker(rank, world, port, kind, dims, chunks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1905_09539_b200.dist import DecoupledSharded
        coeffs, _, rhs = R.baseline_problem(kind, dims, seed=9)
        f = [R.schur(a) for a in coeffs]   # (U, T) per mode, shared setup
        be = CpuDecoupled(rank, world, [t for _, t in f], [u for u, _ in f], chunks)
        lo, hi = be.bd[rank], be.bd[rank + 1]
        b = torch.from_numpy(np.asfortranarray(rhs[..., lo:hi]).reshape(-1, order="F").copy())
        x = torch.zeros_like(b)
        sh = DecoupledSharded(be)
        sh.solve(b, x)
        want = R.solve_laplace(coeffs, rhs, n_min=4)[..., lo:hi]
        got = x.numpy().reshape(want.shape, order="F")
        err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
        q.put((rank, lo, hi, be.b0, err, be.cb))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,kind,dims,chunks", [
    (2, 2, (8, 6, 10), 1), (3, 2, (9, 5, 12), 1), (2, 1, (8, 7, 6), 1), (3, 2, (6, 4, 3, 9), 1),
    # pipelined exchanges: 2-4 chunks per slab (ragged, and more chunks than some slabs have cells)
    (2, 2, (8, 6, 10), 2), (3, 2, (9, 5, 12), 3), (2, 2, (7, 5, 9), 4), (3, 2, (6, 4, 3, 9), 2)])
def test_decoupled_sharded_gloo(world, kind, dims, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, dims, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == 0 and res[-1][2] == dims[-1]
    b0 = res[0][3]
    assert b0[0] == 0 and b0[-1] == dims[0] and all(b1 > a1 for a1, b1 in zip(b0, b0[1:]))
    for r, lo, hi, _, err, cb in res:
        assert hi > lo
        assert err < 1e-10, (r, err)
        assert len(cb) == chunks + 1 and cb[0] == 0 and cb[-1] == hi - lo
        assert all(b1 >= a1 for a1, b1 in zip(cb, cb[1:]))
