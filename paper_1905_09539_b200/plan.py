"""Device-resident plans (tsg_plan_*): the bench and multi-run callers set a
problem up once (factors uploaded, tiles and schedule built) and execute it
many times on buffers that already live in HBM (torch CUDA tensors), or with
host buffers (H2D/D2H inside the call)."""
from __future__ import annotations

import ctypes

import numpy as np

from ._lib import TsgOpts, TsgReport, c_dbl_p, c_dbl_pp, lib
from .api import _f, _ptr, _ptrs, gpu_error


class Context:
    def __init__(self, device: int = 0):
        self.h = ctypes.c_void_p()
        dev = (ctypes.c_int * 1)(device)
        rc = lib().tsg_create(1, dev, ctypes.byref(self.h))
        if rc != 0:
            raise gpu_error(f"tsg_create failed ({rc})")

    def stream_ptr(self) -> int:
        return int(lib().tsg_ctx_stream(self.h) or 0)

    def error(self) -> str:
        return lib().tsg_last_error(self.h).decode()

    def close(self):
        if self.h:
            lib().tsg_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        self.close()


class Plan:
    """family 0: Laplace with (T, U) per mode; family 1: gsylv with T[0]=S,
    U[0]=Q and the extra Tc, Z factors."""

    def __init__(self, ctx: Context, family: int, T: list, U: list | None, Tc=None, Z=None,
                 reduced_only: bool = False, n_min: int = 0, tile=None, skip_transform=(),
                 free_mode: int = -1):
        """skip_transform: modes whose transforms are the identity (their U
        entry may be None); free_mode: the decoupled solve's free mode (-1:
        the plan's choice).  Both serve the slab-sharded solve (dist.py)."""
        self.ctx = ctx
        self.T = [_f(t) for t in T]
        self.U = [(_f(u) if u is not None else np.zeros((1, 1), order="F")) for u in U] if U is not None else None
        self.Tc = _f(Tc) if Tc is not None else None
        self.Z = _f(Z) if Z is not None else None
        self.dims = [t.shape[0] for t in self.T]
        d = len(self.dims)
        opts = TsgOpts()
        lib().tsg_default_opts(ctypes.byref(opts))
        opts.n_min = n_min
        opts.skip_transform_mask = sum(1 << int(m) for m in skip_transform)
        opts.free_mode = int(free_mode)
        if tile:
            for m, b in enumerate(tile):
                opts.tile[m] = int(b)
        tp, k1 = _ptrs(self.T)
        if self.U is not None:
            up, k2 = _ptrs(self.U)
        else:
            up = ctypes.cast((c_dbl_p * d)(), c_dbl_pp)
        self.h = ctypes.c_void_p()
        rc = lib().tsg_plan_create(ctx.h, family, d, (ctypes.c_int * d)(*self.dims), tp, up,
                                   _ptr(self.Tc) if self.Tc is not None else None,
                                   _ptr(self.Z) if self.Z is not None else None,
                                   1 if reduced_only else 0, ctypes.byref(opts),
                                   ctypes.byref(self.h))
        if rc != 0:
            raise gpu_error(f"tsg_plan_create failed ({rc}): {ctx.error()}")
        self.n = int(np.prod(self.dims))

    def free_mode(self) -> int:
        """Free mode of the eigen-decoupled solve (-1: tile-DAG kernels)."""
        return int(lib().tsg_plan_free_mode(self.h))

    def transform(self, direction: int, in_ptr: int, out_ptr: int, stream: int = 0) -> None:
        """Transforms only (0 forward, 1 back), device buffers, on `stream`."""
        rc = lib().tsg_plan_transform(self.h, int(direction), ctypes.c_void_p(in_ptr), ctypes.c_void_p(out_ptr),
                                      ctypes.c_void_p(stream))
        if rc != 0:
            raise gpu_error(f"tsg_plan_transform failed ({rc}): {self.ctx.error()}")

    def info(self):
        nt = ctypes.c_int64()
        ext = (ctypes.c_int * 8)()
        fa = ctypes.c_double()
        lib().tsg_plan_info(self.h, ctypes.byref(nt), ext, ctypes.byref(fa))
        return dict(n_tiles=nt.value, tile=list(ext)[:len(self.dims)], flops_alg=fa.value)

    def describe(self) -> str:
        """The reduced-solve kernel this plan runs (tsg_plan_describe)."""
        buf = ctypes.create_string_buffer(160)
        lib().tsg_plan_describe(self.h, buf, 160)
        return buf.value.decode()

    def execute_device(self, b_ptr: int, x_ptr: int) -> TsgReport:
        rep = TsgReport()
        rc = lib().tsg_plan_execute(self.h, ctypes.c_void_p(b_ptr), ctypes.c_void_p(x_ptr), 1,
                                    ctypes.byref(rep))
        if rc != 0:
            raise gpu_error(f"tsg_plan_execute failed ({rc}): {self.ctx.error()}")
        return rep

    def enqueue_device(self, b_ptr: int, x_ptr: int) -> None:
        """Asynchronous solve on the context stream (tsg_plan_enqueue)."""
        rc = lib().tsg_plan_enqueue(self.h, ctypes.c_void_p(b_ptr), ctypes.c_void_p(x_ptr))
        if rc != 0:
            raise gpu_error(f"tsg_plan_enqueue failed ({rc}): {self.ctx.error()}")

    def set_serial(self, serial: bool) -> None:
        """Every kernel after its predecessor (tsg_plan_set_serial): the
        per-phase times of execute_* become per-kernel launch times."""
        rc = lib().tsg_plan_set_serial(self.h, 1 if serial else 0)
        if rc != 0:
            raise gpu_error(f"tsg_plan_set_serial failed ({rc}): {self.ctx.error()}")

    def sync(self) -> TsgReport:
        """Wait for every enqueued solve (tsg_plan_sync); zero pivot of the last."""
        rep = TsgReport()
        rc = lib().tsg_plan_sync(self.h, ctypes.byref(rep))
        if rc != 0:
            raise gpu_error(f"tsg_plan_sync failed ({rc}): {self.ctx.error()}")
        return rep

    def execute_host(self, b: np.ndarray, x: np.ndarray) -> TsgReport:
        rep = TsgReport()
        rc = lib().tsg_plan_execute(self.h, b.ctypes.data_as(ctypes.c_void_p),
                                    x.ctypes.data_as(ctypes.c_void_p), 0, ctypes.byref(rep))
        if rc != 0:
            raise gpu_error(f"tsg_plan_execute failed ({rc}): {self.ctx.error()}")
        return rep

    def execute_stream(self, b_ptrs: list, x_ptrs: list) -> TsgReport:
        """Solve len(b_ptrs) right-hand sides from HOST buffers (raw pointers,
        pinned memory recommended) with copy/compute overlap
        (tsg_plan_execute_stream)."""
        n = len(b_ptrs)
        if len(x_ptrs) != n:
            raise ValueError("execute_stream: as many outputs as inputs")
        bp = (ctypes.c_void_p * max(n, 1))(*[ctypes.c_void_p(int(p)) for p in b_ptrs])
        xp = (ctypes.c_void_p * max(n, 1))(*[ctypes.c_void_p(int(p)) for p in x_ptrs])
        rep = TsgReport()
        rc = lib().tsg_plan_execute_stream(self.h, n, bp, xp, ctypes.byref(rep))
        if rc != 0:
            raise gpu_error(f"tsg_plan_execute_stream failed ({rc}): {self.ctx.error()}")
        return rep

    def close(self):
        if self.h:
            lib().tsg_plan_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        self.close()
