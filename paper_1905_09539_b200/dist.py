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


def chunk_bounds(T_last: np.ndarray, bd: list[int], chunks: int) -> list[list[int]]:
    """Per rank, the bounds (chunks + 1, relative to the slab start) of the
    pipeline chunks of its last-mode slab: balanced, never inside a 2x2 cell
    of T_last (so every chunk is a valid sub-problem shape), possibly empty
    when the slab has fewer cells than chunks.  Every rank computes the table
    for all ranks (the receive side of the all-to-alls needs it)."""
    T_last = _f(T_last)
    out = []
    for r in range(len(bd) - 1):
        lo, hi = bd[r], bd[r + 1]
        if chunks <= 1 or hi - lo <= 1:
            out.append([0] + [hi - lo] * max(chunks, 1))
            continue
        cuts = [0]
        for c in range(1, chunks):
            t = max(cuts[-1], min(hi - lo, round(c * (hi - lo) / chunks)))
            if 0 < t < hi - lo and T_last[lo + t, lo + t - 1] != 0.0:
                t += 1  # not inside a 2x2 cell
            cuts.append(min(t, hi - lo))
        out.append(cuts + [hi - lo])
    return out


class DeviceDecoupled:
    """CUDA backend of DecoupledSharded for one rank (the phase-B plan and one
    phase-A plan per distinct chunk extent)."""

    def __init__(self, ctx, rank: int, nranks: int, T: list, U: list, f: int | None = None, chunks: int = 1):
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
        # phase A runs per pipeline chunk of the slab (chunks = 1: the slab);
        # the last mode is not transformed there, so a plan serves every chunk
        # of its extent
        self.cb_all = chunk_bounds(self.T[-1], self.bd, chunks)
        self.cb = self.cb_all[rank]
        self.plans_a = {}
        for c in range(len(self.cb) - 1):
            c0, c1 = lo + self.cb[c], lo + self.cb[c + 1]
            if c1 - c0 <= 0 or c1 - c0 in self.plans_a:
                continue
            ta = self.T[:-1] + [np.asfortranarray(self.T[-1][c0:c1, c0:c1])]
            self.plans_a[c1 - c0] = Plan(ctx, 0, ta, self.U[:-1] + [None], skip_transform=(d - 1,),
                                         free_mode=self.f)
        self.plan_a = self.plans_a.get(hi - lo)  # the whole-slab plan (chunks = 1)
        for p, nm in [(self.plan_b, "B")] + [(q, "A") for q in self.plans_a.values()]:
            if p.free_mode() != self.f:
                raise gpu_error(f"sharded decoupled solve: phase-{nm} plan not decoupled along mode {self.f} "
                                f"({p.describe()})")
        self.slab_elems = int(np.prod(self.dims[:-1]))
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.stream = ctx.stream_ptr()

    def empty(self, n: int):
        import torch
        return torch.empty(int(n), dtype=torch.float64, device=self.dev)

    def _a(self, direction: int, src, dst) -> None:
        """Phase-A transforms of a whole slab or of one chunk (the extent
        follows from the buffer length)."""
        rows = src.numel() // self.slab_elems
        if rows in self.plans_a:
            self.plans_a[rows].transform(direction, src.data_ptr(), dst.data_ptr(), self.stream)
            return
        # a whole slab handed to a chunked backend: chunk by chunk
        if rows != self.bd[self.rank + 1] - self.bd[self.rank]:
            raise gpu_error(f"sharded decoupled solve: no phase-A plan for {rows} last-mode rows")
        for c in range(len(self.cb) - 1):
            e0, e1 = self.cb[c] * self.slab_elems, self.cb[c + 1] * self.slab_elems
            if e1 > e0:
                self._a(direction, src[e0:e1], dst[e0:e1])

    def a_forward(self, b, out) -> None:
        self._a(0, b, out)

    def a_back(self, x, out) -> None:
        self._a(1, x, out)

    def b_solve(self, z, out) -> None:
        self.plan_b.enqueue_device(z.data_ptr(), out.data_ptr())

    def repack(self, src, dst, unpack: bool) -> None:
        """Re-sharding pack (runs of n0 -> per-peer mode-0 column segments, the
        all-to-all send layout) or unpack of one slab / chunk on the device
        (tsg_slab_pack, the library's own kernel), on the backend's stream."""
        n0 = self.dims[0]
        b0 = (ctypes.c_int * (self.nranks + 1))(*self.b0)
        rc = lib().tsg_slab_pack(self.ctx.h, ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
                                 src.numel() // n0, n0, self.nranks, b0, 1 if unpack else 0,
                                 ctypes.c_void_p(self.stream))
        if rc != 0:
            raise gpu_error(f"tsg_slab_pack failed ({rc}): {self.ctx.last_error()}")

    def check(self) -> None:
        rep = self.plan_b.sync()
        if rep.zero_pivot_index >= 0:
            raise gpu_error(f"sharded decoupled solve: singular base cell ({rep.zero_pivot_index})")

    def close(self):
        for p in list(getattr(self, "plans_a", {}).values()) + [getattr(self, "plan_b", None)]:
            if p is not None:
                p.close()
        self.plans_a = {}
        self.plan_a = self.plan_b = None


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
        backend's device; everything is ordered on the backend's stream.
        With a chunked backend (DeviceDecoupled(chunks=K)) the slab is
        pipelined in K pieces along the last mode: chunk c's all-to-all runs
        on the communication stream while chunk c + 1 is transformed (and, on
        the way back, chunk c is back-transformed while chunk c + 1 is still
        in flight), so only ~1/K of each exchange is exposed."""
        be = self.be
        if len(getattr(be, "cb", [0, 0])) > 2:
            return self._solve_chunked(b, x, check)
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
        if hasattr(be, "repack"):
            be.repack(self.ya, self.sa, False)
        else:
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
        if hasattr(be, "repack"):
            be.repack(self.ra, self.ya, True)
        else:
            self._run_torch(unpack)
        be.a_back(self.ya, x)
        if check and hasattr(be, "check"):
            be.check()
        return x

    # -- chunked pipeline -------------------------------------------------
    def _chunk_views(self, c: int):
        """Per peer q, the views that chunk c exchanges with q: `mine[q]` in
        the packed send/receive slot of this rank's chunk c (blocks
        (rows_c, mid, Q_q) in rank order inside the chunk's piece of sa / ra)
        and `theirs[q]` = the rows of q's chunk c inside block q of the
        phase-B buffers zb / xb (block q is (R_q, mid, Q_r): its chunk rows
        are contiguous)."""
        be = self.be
        r, P = be.rank, be.nranks
        r0 = self.rows_0[r]
        rows_c = be.cb[c + 1] - be.cb[c]
        e0 = be.cb[c] * self.mid * be.dims[0]
        mine, o = [], e0
        for q in range(P):
            k = rows_c * self.mid * self.rows_0[q]
            mine.append((o, o + k))
            o += k
        theirs, blk = [], 0
        for q in range(P):
            cq0, cq1 = be.cb_all[q][c], be.cb_all[q][c + 1]
            theirs.append((blk + cq0 * self.mid * r0, blk + cq1 * self.mid * r0))
            blk += self.rows_d[q] * self.mid * r0
        return mine, theirs

    def _exchange(self, out, out_rng, inp, in_rng, comm, after):
        """All-to-all of the given (start, stop) pieces: inp[in_rng[q]] -> rank
        q, out[out_rng[q]] <- rank q.  CUDA: list-based NCCL all_to_all
        straight between the views, asynchronous on the communication stream
        once `after` (an event of the compute stream) has fired; returns the
        callable that makes the compute stream wait for it.  CPU (gloo, tests):
        all_to_all_single through contiguous staging, completed on return."""
        import torch
        import torch.distributed as dist
        be = self.be
        outs = [out[a:z] for a, z in out_rng]
        ins = [inp[a:z] for a, z in in_rng]
        if be.nranks == 1 and not (dist.is_available() and dist.is_initialized()):
            self._run_torch(lambda: outs[0].copy_(ins[0]))
            return lambda: None
        if out.is_cuda:
            with torch.cuda.stream(comm):
                comm.wait_event(after)
                work = dist.all_to_all(outs, ins, group=self.group, async_op=True)
            return work.wait  # called under the compute stream: a stream-side wait
        stage_in = torch.cat(ins) if ins else inp[:0]
        stage_out = torch.empty(sum(z - a for a, z in out_rng), dtype=out.dtype)
        dist.all_to_all_single(stage_out, stage_in, [z - a for a, z in out_rng], [z - a for a, z in in_rng],
                               group=self.group)
        o = 0
        for v in outs:
            v.copy_(stage_out[o:o + v.numel()])
            o += v.numel()
        return lambda: None

    def _solve_chunked(self, b, x, check: bool = False):
        import torch
        be = self.be
        P, n0 = be.nranks, be.dims[0]
        K = len(be.cb) - 1
        cuda = self.ya.is_cuda
        if cuda:
            compute = torch.cuda.ExternalStream(be.stream, device=self.ya.device)
            if getattr(self, "_comm", None) is None:
                self._comm = torch.cuda.Stream(device=self.ya.device)
            comm = self._comm
        else:
            compute = comm = None

        def on_compute(fn):
            if cuda:
                with torch.cuda.stream(compute):
                    return fn()
            return fn()

        def mark():
            if not cuda:
                return None
            ev = torch.cuda.Event()
            ev.record(compute)
            return ev

        views = [self._chunk_views(c) for c in range(K)]
        slab = self.mid * n0
        # forward: transform + pack chunk c, then its exchange overlaps chunk c + 1
        waits = []
        for c in range(K):
            rows_c = be.cb[c + 1] - be.cb[c]
            e0, e1 = be.cb[c] * slab, be.cb[c + 1] * slab
            mine, theirs = views[c]
            if rows_c > 0:
                be.a_forward(b[e0:e1], self.ya[e0:e1])

                def pack(rows_c=rows_c, e0=e0, e1=e1, mine=mine):
                    v = self.ya[e0:e1].view(rows_c, self.mid, n0)
                    for q in range(P):
                        a, z = mine[q]
                        self.sa[a:z].view(rows_c, self.mid, self.rows_0[q]).copy_(v[:, :, be.b0[q]:be.b0[q + 1]])
                if hasattr(be, "repack"):
                    be.repack(self.ya[e0:e1], self.sa[e0:e1], False)
                else:
                    on_compute(pack)
            waits.append(self._exchange(self.zb, theirs, self.sa, mine, comm, mark()))
        for w in waits:
            on_compute(w)
        be.b_solve(self.zb, self.xb)
        # back: every chunk's exchange is queued behind the solve; chunk c is
        # unpacked and back-transformed as soon as it has landed
        done = mark()
        waits = [self._exchange(self.ra, views[c][0], self.xb, views[c][1], comm, done) for c in range(K)]
        for c in range(K):
            rows_c = be.cb[c + 1] - be.cb[c]
            e0, e1 = be.cb[c] * slab, be.cb[c + 1] * slab
            mine = views[c][0]
            on_compute(waits[c])
            if rows_c == 0:
                continue

            def unpack(rows_c=rows_c, e0=e0, e1=e1, mine=mine):
                v = self.ya[e0:e1].view(rows_c, self.mid, n0)
                for q in range(P):
                    a, z = mine[q]
                    v[:, :, be.b0[q]:be.b0[q + 1]].copy_(self.ra[a:z].view(rows_c, self.mid, self.rows_0[q]))
            if hasattr(be, "repack"):
                be.repack(self.ra[e0:e1], self.ya[e0:e1], True)
            else:
                on_compute(unpack)
            be.a_back(self.ya[e0:e1], x[e0:e1])
        if cuda:
            # the next solve's first pack overwrites sa: it must not pass the
            # exchanges still reading it (they completed before b_solve), and
            # the communication stream must not run ahead of this solve
            comm.wait_event(mark())
        if check and hasattr(be, "check"):
            be.check()
        return x


def decoupled_emulated_solve(ctx, T: list, U: list, b_full: np.ndarray, nslabs: int, chunks: int = 1) -> np.ndarray:
    """All slabs of the sharded decoupled solve in one process on one GPU:
    the same plans and pack/unpack as the ranks, the all-to-alls done by
    copies between the slabs' buffers (validation on a single device).
    chunks > 1: phase A runs on the per-chunk plans of the pipelined solve."""
    import torch
    dims = [t.shape[0] for t in T]
    d = len(dims)
    bes = [DeviceDecoupled(ctx, r, nslabs, T, U, chunks=chunks) for r in range(nslabs)]
    sh = [DecoupledSharded(be) for be in bes]
    bd, b0 = bes[0].bd, bes[0].b0
    st = torch.cuda.ExternalStream(ctx.stream_ptr())
    with torch.cuda.stream(st):
        bs = [torch.from_numpy(np.ascontiguousarray(b_full[..., bd[r]:bd[r + 1]]).reshape(-1, order="F")).cuda()
              for r in range(nslabs)]
        xs = [torch.empty_like(v) for v in bs]
        for r in range(nslabs):
            bes[r].a_forward(bs[r], sh[r].ya)
            bes[r].repack(sh[r].ya, sh[r].sa, False)  # the library's pack kernel, as on the ranks
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
            bes[r].repack(sh[r].ra, sh[r].ya, True)
            bes[r].a_back(sh[r].ya, xs[r])
        torch.cuda.synchronize()
    for be in bes:
        be.check()
    parts = [xs[r].cpu().numpy().reshape(tuple(dims[:-1]) + (bd[r + 1] - bd[r],), order="F")
             for r in range(nslabs)]
    for be in bes:
        be.close()
    return np.concatenate(parts, axis=d - 1)
