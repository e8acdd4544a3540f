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
