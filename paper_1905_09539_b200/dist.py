"""Slab-sharded multi-GPU Laplace solve, one process per GPU.

The tensor is cut into slabs along its last mode (tile-aligned; a slab is a
contiguous piece of the column-major tensor, so rank r holds ``B[..., lo_r:hi_r]``).
One solve is the step sequence of the C-ABI (include/tsylv_gpu.h, tsg_dplan_*):

    forward_local   B_r x_m U_m^T for m < d-1             (slab-local DMMA GEMMs)
    all-gather      send slots -> gather buffer            (torch.distributed / NCCL)
    forward_split   gather x_{d-1} U_{d-1}^T[R_r, :]       -> B~_r
    solve           dataflow kernel over the rank's tiles, reading the other
                    ranks' tiles and flags through CUDA IPC peer mappings
    back_local, all-gather, back_split                     -> X_r

``ShardedLaplace`` is the orchestration; the device steps come from a backend:
``DeviceSlabs`` (the CUDA library, the product path) or, in tests, a CPU stand-in
that follows the same step semantics (tests/test_dist_gloo.py).  With
``emulate=True`` one process owns every slab on one GPU and the collectives
disappear (the gather buffer doubles as the send slots); this validates the
sharded kernels and addressing on a single device.
"""
from __future__ import annotations

import ctypes

import numpy as np

from ._lib import TsgOpts, c_dbl_pp, lib
from .api import _f, _ptrs, gpu_error

IPC_BYTES = 128


def slab_bounds(n: int, T: np.ndarray, nranks: int, tile: int = 8) -> list[int]:
    """Row bounds (nranks + 1) of the slabs along a mode of extent n with
    quasi-triangular factor T: tile-aligned, never inside a 2x2 block, balanced."""
    T = _f(T)
    out = (ctypes.c_int * (nranks + 1))()
    rc = lib().tsg_slab_bounds(n, T.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), tile, nranks, out)
    if rc != 0:
        raise ValueError(f"tsg_slab_bounds failed ({rc}): {nranks} slabs of extent {n}")
    return list(out)


class _CudaView:
    """Zero-copy torch view of a raw device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3}


def device_view(ptr: int, n: int, device):
    import torch
    return torch.as_tensor(_CudaView(ptr, n), device=device)


class DeviceSlabs:
    """The CUDA backend: one tsg_dplan (this rank's slab, or all slabs when
    emulated) on the context's device."""

    def __init__(self, ctx, rank: int, nranks: int, T: list, U: list, emulate: bool = False,
                 tile=None):
        import torch
        self.ctx = ctx
        self.rank, self.nranks, self.emulate = rank, nranks, emulate
        self.T = [_f(t) for t in T]
        self.U = [_f(u) for u in U]
        self.dims = [t.shape[0] for t in self.T]
        d = len(self.dims)
        opts = TsgOpts()
        lib().tsg_default_opts(ctypes.byref(opts))
        if tile:
            for m, b in enumerate(tile):
                opts.tile[m] = int(b)
        tp, _k1 = _ptrs(self.T)
        up, _k2 = _ptrs(self.U)
        self.h = ctypes.c_void_p()
        rc = lib().tsg_dplan_create(ctx.h, rank, nranks, 1 if emulate else 0, d,
                                    (ctypes.c_int * d)(*self.dims), tp, up, ctypes.byref(opts),
                                    ctypes.byref(self.h))
        if rc != 0:
            raise gpu_error(f"tsg_dplan_create failed ({rc}): {ctx.error()}")
        bounds = (ctypes.c_int * (nranks + 1))()
        se, sn = ctypes.c_int64(), ctypes.c_int64()
        lib().tsg_dplan_info(self.h, bounds, ctypes.byref(se), ctypes.byref(sn))
        self.bounds = list(bounds)
        self.slab_elems, self.send_elems = se.value, sn.value
        send, gath = ctypes.c_void_p(), ctypes.c_void_p()
        lib().tsg_dplan_buffers(self.h, ctypes.byref(send), ctypes.byref(gath))
        dev = torch.device("cuda", torch.cuda.current_device())
        self.gather = device_view(gath.value, self.send_elems * nranks, dev)
        self.send = None if emulate else device_view(send.value, self.send_elems, dev)

    # ---- IPC peer mappings (multi-GPU) ----
    def ipc_handles(self) -> bytes:
        buf = ctypes.create_string_buffer(IPC_BYTES)
        self._check(lib().tsg_dplan_ipc_export(self.h, buf), "ipc_export")
        return buf.raw

    def ipc_open(self, handles: list[bytes]) -> None:
        allh = ctypes.create_string_buffer(b"".join(handles), IPC_BYTES * self.nranks)
        self._check(lib().tsg_dplan_ipc_import(self.h, allh), "ipc_import")

    # ---- steps (enqueued on `stream`, a cudaStream_t as int) ----
    def forward_local(self, b, stream: int) -> None:
        self._check(lib().tsg_dplan_forward_local(self.h, ctypes.c_void_p(b.data_ptr()),
                                                  ctypes.c_void_p(stream)), "forward_local")

    def forward_split(self, stream: int) -> None:
        self._check(lib().tsg_dplan_forward_split(self.h, ctypes.c_void_p(stream)), "forward_split")

    def solve(self, stream: int, group=None) -> None:
        self._check(lib().tsg_dplan_solve(self.h, ctypes.c_void_p(stream)), "solve")

    def back_local(self, stream: int) -> None:
        self._check(lib().tsg_dplan_back_local(self.h, ctypes.c_void_p(stream)), "back_local")

    def back_split(self, x, stream: int) -> None:
        self._check(lib().tsg_dplan_back_split(self.h, ctypes.c_void_p(x.data_ptr()),
                                               ctypes.c_void_p(stream)), "back_split")

    def status(self, stream: int) -> None:
        self._check(lib().tsg_dplan_status(self.h, ctypes.c_void_p(stream)), "status")

    def _check(self, rc: int, what: str) -> None:
        if rc != 0:
            raise gpu_error(f"tsg_dplan_{what} failed ({rc}): {self.ctx.error()}")

    def close(self):
        if getattr(self, "h", None):
            lib().tsg_dplan_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


class ShardedLaplace:
    """Orchestrates one sharded solve per call.

    backend: DeviceSlabs (or a test stand-in with the same methods and
    ``bounds``, ``send``, ``gather`` attributes); group: torch.distributed
    process group (None = default) for the all-gathers; ignored when the
    backend is emulated.
    """

    def __init__(self, backend, group=None):
        self.be = backend
        self.group = group
        self.emulate = backend.emulate
        if not self.emulate and hasattr(backend, "ipc_handles"):
            import torch.distributed as dist
            mine = backend.ipc_handles()
            allh = [None] * backend.nranks
            dist.all_gather_object(allh, mine, group=group)
            backend.ipc_open(allh)
            dist.barrier(group=group)

    def _all_gather(self, stream):
        """NCCL all-gather of the send slots, ordered on `stream`: torch
        enqueues the collective behind its *current* stream and makes that
        stream wait for it, so the library's stream is made current for the
        call (the gather must see forward_local's output, and forward_split
        must see the gathered data)."""
        import torch
        import torch.distributed as dist
        if self.be.gather.is_cuda:
            with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=self.be.gather.device)):
                dist.all_gather_into_tensor(self.be.gather, self.be.send, group=self.group)
        else:
            dist.all_gather_into_tensor(self.be.gather, self.be.send, group=self.group)

    def solve(self, b, x, stream: int | None = None, check: bool = False):
        """b, x: this rank's slab (the whole tensor when emulated) as flat
        column-major tensors on the backend's device; enqueued on `stream`
        (a cudaStream_t as int; default: torch's current stream, so inputs
        written by torch are ordered before the solve)."""
        be = self.be
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream if b.is_cuda else 0
        be.forward_local(b, stream)
        if not self.emulate:
            self._all_gather(stream)
        be.forward_split(stream)
        be.solve(stream, self.group)
        be.back_local(stream)
        if not self.emulate:
            self._all_gather(stream)
        be.back_split(x, stream)
        if check:
            be.status(stream)
        return x


# ---------------------------------------------------------------------------
# Eigen-decoupled slab sharding: the default multi-GPU path.
#
# Every mode but the free mode f is in its eigenbasis after the transforms,
# so the solve couples elements only along f.  Ranks hold slabs along the
# LAST mode (input and output layout, R_r); the solve runs on slabs along
# MODE 0 (Q_r, whole 2x2 cells), where every fibre along f and every mode-(d-1)
# fibre is complete.  Per solve:
#
#   A  forward transforms of modes 0..d-2 on the last-mode slab   (local)
#      all-to-all: last-mode slabs -> mode-0 slabs               (NCCL)
#   B  forward transform of mode d-1, fibre solve along f,
#      back transform of mode d-1 on the mode-0 slab              (local)
#      all-to-all: mode-0 slabs -> last-mode slabs                (NCCL)
#   C  back transforms of modes 0..d-2                            (local)
#
# Each all-to-all moves 8 N (P-1) / P^2 bytes per rank (a slab's share of
# every other rank's slab), against 8 N (P-1) / P for an all-gather of the
# whole tensor.  Phase A/C and phase B are tsg plans on the two slab shapes
# (skip_transform / free_mode options); the receive buffer of the first
# all-to-all is already the column-major mode-0 slab (the last mode is the
# slowest), and the second all-to-all sends the phase-B result as is.
# ---------------------------------------------------------------------------


def decoupled_free_mode(dims) -> int:
    """Free mode of the sharded decoupled solve (CPU stand-in rule): the
    shortest of modes 1..d-1 (mode 0, the solve-phase shard mode, must be an
    eigen mode).  The CUDA backend takes the plan's own choice."""
    d = len(dims)
    if d < 2:
        raise ValueError("the sharded decoupled solve needs d >= 2")
    return min(range(1, d), key=lambda m: (dims[m], m))


class DeviceDecoupled:
    """CUDA backend of DecoupledSharded for one rank (two tsg plans)."""

    def __init__(self, ctx, rank: int, nranks: int, T: list, U: list, f: int | None = None):
        import torch
        from .plan import Plan
        self.ctx, self.rank, self.nranks = ctx, rank, nranks
        self.T = [_f(t) for t in T]
        self.U = [_f(u) for u in U]
        self.dims = [t.shape[0] for t in self.T]
        d = len(self.dims)
        if d < 3:
            raise ValueError("the sharded decoupled solve needs d >= 3")
        self.bd = slab_bounds(self.dims[-1], self.T[-1], nranks, tile=1)  # last-mode slabs
        self.b0 = slab_bounds(self.dims[0], self.T[0], nranks, tile=1)    # mode-0 slabs
        # phase B first: its plan picks the free mode (f >= 1, the single-GPU
        # rule), which phase A then follows
        q0, q1 = self.b0[rank], self.b0[rank + 1]
        tb = [np.asfortranarray(self.T[0][q0:q1, q0:q1])] + self.T[1:]
        self.plan_b = Plan(ctx, 0, tb, [None] * (d - 1) + [self.U[-1]], skip_transform=tuple(range(d - 1)),
                           free_mode=-1 if f is None else f)
        self.f = self.plan_b.free_mode()
        if self.f < 1:
            raise gpu_error(f"sharded decoupled solve: phase-B plan not decoupled ({self.plan_b.describe()})")
        lo, hi = self.bd[rank], self.bd[rank + 1]
        ta = self.T[:-1] + [np.asfortranarray(self.T[-1][lo:hi, lo:hi])]
        self.plan_a = Plan(ctx, 0, ta, self.U[:-1] + [None], skip_transform=(d - 1,), free_mode=self.f)
        for p, nm in ((self.plan_a, "A"), (self.plan_b, "B")):
            if p.free_mode() != self.f:
                raise gpu_error(f"sharded decoupled solve: phase-{nm} plan not decoupled along mode {self.f} "
                                f"({p.describe()})")
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.stream = ctx.stream_ptr()

    def empty(self, n: int):
        import torch
        return torch.empty(int(n), dtype=torch.float64, device=self.dev)

    def a_forward(self, b, out) -> None:
        self.plan_a.transform(0, b.data_ptr(), out.data_ptr(), self.stream)

    def a_back(self, x, out) -> None:
        self.plan_a.transform(1, x.data_ptr(), out.data_ptr(), self.stream)

    def b_solve(self, z, out) -> None:
        self.plan_b.enqueue_device(z.data_ptr(), out.data_ptr())

    def check(self) -> None:
        rep = self.plan_b.sync()
        if rep.zero_pivot_index >= 0:
            raise gpu_error(f"sharded decoupled solve: singular base cell ({rep.zero_pivot_index})")

    def close(self):
        for p in (getattr(self, "plan_a", None), getattr(self, "plan_b", None)):
            if p is not None:
                p.close()


class DecoupledSharded:
    """Orchestration of one sharded decoupled Laplace solve per call.

    backend: DeviceDecoupled (CUDA, the product path) or a test stand-in with
    the same attributes (rank, nranks, dims, bd, b0, a_forward, b_solve,
    a_back, empty, stream); group: torch.distributed process group."""

    def __init__(self, backend, group=None):
        self.be = backend
        self.group = group
        be = backend
        d = len(be.dims)
        self.mid = int(np.prod(be.dims[1:d - 1]))
        r, P = be.rank, be.nranks
        self.rows_d = [be.bd[q + 1] - be.bd[q] for q in range(P)]
        self.rows_0 = [be.b0[q + 1] - be.b0[q] for q in range(P)]
        rd, r0 = self.rows_d[r], self.rows_0[r]
        # all-to-all 1: to rank q the block (rows Q_q of mode 0) x mid x R_r
        self.send1 = [self.rows_0[q] * self.mid * rd for q in range(P)]
        self.recv1 = [r0 * self.mid * self.rows_d[q] for q in range(P)]
        self.n_a = be.dims[0] * self.mid * rd
        self.n_b = r0 * self.mid * be.dims[-1]
        self.ya = be.empty(self.n_a)
        self.sa = be.empty(self.n_a)
        self.zb = be.empty(self.n_b)
        self.xb = be.empty(self.n_b)
        self.ra = be.empty(self.n_a)

    def _a2a(self, out, inp, out_sizes, in_sizes):
        import torch
        import torch.distributed as dist
        if self.be.nranks == 1:
            self._run_torch(lambda: out.copy_(inp))
            return
        if out.is_cuda:
            with torch.cuda.stream(torch.cuda.ExternalStream(self.be.stream, device=out.device)):
                dist.all_to_all_single(out, inp, out_sizes, in_sizes, group=self.group)
        else:
            dist.all_to_all_single(out, inp, out_sizes, in_sizes, group=self.group)

    def _run_torch(self, fn):
        import torch
        if self.ya.is_cuda:
            with torch.cuda.stream(torch.cuda.ExternalStream(self.be.stream, device=self.ya.device)):
                fn()
        else:
            fn()

    def solve(self, b, x, check: bool = False):
        """b, x: this rank's last-mode slab (flat, column-major), on the
        backend's device; everything is ordered on the backend's stream."""
        be = self.be
        P, n0 = be.nranks, be.dims[0]
        rd = self.rows_d[be.rank]
        be.a_forward(b, self.ya)
        # pack: ya as row-major (R_r, mid, n0) -> blocks [:, :, Q_q] in rank order

        def pack():
            v = self.ya.view(rd, self.mid, n0)
            o = 0
            for q in range(P):
                k = self.send1[q]
                self.sa[o:o + k].view(rd, self.mid, self.rows_0[q]).copy_(v[:, :, be.b0[q]:be.b0[q + 1]])
                o += k
        self._run_torch(pack)
        self._a2a(self.zb, self.sa, self.recv1, self.send1)
        be.b_solve(self.zb, self.xb)
        self._a2a(self.ra, self.xb, self.send1, self.recv1)

        def unpack():
            v = self.ya.view(rd, self.mid, n0)
            o = 0
            for q in range(P):
                k = self.send1[q]
                v[:, :, be.b0[q]:be.b0[q + 1]].copy_(self.ra[o:o + k].view(rd, self.mid, self.rows_0[q]))
                o += k
        self._run_torch(unpack)
        be.a_back(self.ya, x)
        if check and hasattr(be, "check"):
            be.check()
        return x


def decoupled_emulated_solve(ctx, T: list, U: list, b_full: np.ndarray, nslabs: int) -> np.ndarray:
    """All slabs of the sharded decoupled solve in one process on one GPU:
    the same plans and pack/unpack as the ranks, the all-to-alls done by
    copies between the slabs' buffers (validation on a single device)."""
    import torch
    dims = [t.shape[0] for t in T]
    d = len(dims)
    bes = [DeviceDecoupled(ctx, r, nslabs, T, U) for r in range(nslabs)]
    sh = [DecoupledSharded(be) for be in bes]
    bd, b0 = bes[0].bd, bes[0].b0
    st = torch.cuda.ExternalStream(ctx.stream_ptr())
    with torch.cuda.stream(st):
        bs = [torch.from_numpy(np.ascontiguousarray(b_full[..., bd[r]:bd[r + 1]]).reshape(-1, order="F")).cuda()
              for r in range(nslabs)]
        xs = [torch.empty_like(v) for v in bs]
        for r in range(nslabs):
            bes[r].a_forward(bs[r], sh[r].ya)
            v = sh[r].ya.view(sh[r].rows_d[r], sh[r].mid, dims[0])
            o = 0
            for q in range(nslabs):
                k = sh[r].send1[q]
                sh[r].sa[o:o + k].view(sh[r].rows_d[r], sh[r].mid, sh[r].rows_0[q]).copy_(v[:, :, b0[q]:b0[q + 1]])
                o += k
        # all-to-all 1: rank q's receive block from r = r's send block for q
        for q in range(nslabs):
            o = 0
            for r in range(nslabs):
                k = sh[q].recv1[r]
                so = sum(sh[r].send1[:q])
                sh[q].zb[o:o + k].copy_(sh[r].sa[so:so + k])
                o += k
        for q in range(nslabs):
            bes[q].b_solve(sh[q].zb, sh[q].xb)
        # all-to-all 2 (the reverse)
        for r in range(nslabs):
            o = 0
            for q in range(nslabs):
                k = sh[r].send1[q]
                so = sum(sh[q].recv1[:r])
                sh[r].ra[o:o + k].copy_(sh[q].xb[so:so + k])
                o += k
        for r in range(nslabs):
            v = sh[r].ya.view(sh[r].rows_d[r], sh[r].mid, dims[0])
            o = 0
            for q in range(nslabs):
                k = sh[r].send1[q]
                v[:, :, b0[q]:b0[q + 1]].copy_(sh[r].ra[o:o + k].view(sh[r].rows_d[r], sh[r].mid, sh[r].rows_0[q]))
                o += k
            bes[r].a_back(sh[r].ya, xs[r])
        torch.cuda.synchronize()
    for be in bes:
        be.check()
    parts = [xs[r].cpu().numpy().reshape(tuple(dims[:-1]) + (bd[r + 1] - bd[r],), order="F")
             for r in range(nslabs)]
    for be in bes:
        be.close()
    return np.concatenate(parts, axis=d - 1)
