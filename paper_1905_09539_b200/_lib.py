"""Loader for the in-tree sm_100a library (fails loudly when it is missing).

There is no CPU fallback anywhere in the product path: every solve entry point
goes through ``libtsylv_gpu.so`` (CUDA kernels + C-ABI + C++ drop-in facade).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtsylv_gpu.so")

_lib = None

c_int_p = ctypes.POINTER(ctypes.c_int)
c_dbl_p = ctypes.POINTER(ctypes.c_double)
c_dbl_pp = ctypes.POINTER(c_dbl_p)


class TsgOpts(ctypes.Structure):
    _fields_ = [("n_min", ctypes.c_int), ("tile", ctypes.c_int * 8),
                ("inputs_on_device", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("skip_transform_mask", ctypes.c_int), ("free_mode", ctypes.c_int)]


class TsgReport(ctypes.Structure):
    _fields_ = [("t_fwd_ms", ctypes.c_double), ("t_solve_ms", ctypes.c_double),
                ("t_back_ms", ctypes.c_double), ("t_h2d_ms", ctypes.c_double),
                ("t_d2h_ms", ctypes.c_double), ("t_total_ms", ctypes.c_double),
                ("flops_alg", ctypes.c_double), ("flops_exec", ctypes.c_double),
                ("zero_pivot_index", ctypes.c_int), ("kernel_launches", ctypes.c_int)]


# Every symbol include/tsylv_gpu.h declares (checked by tests/test_abi.py).
TSG_SYMBOLS = [
    "tsg_default_opts", "tsg_create", "tsg_destroy", "tsg_last_error", "tsg_ctx_stream",
    "tsg_laplace_solve",
    "tsg_laplace_reduced", "tsg_gsylv_solve", "tsg_gsylv_reduced", "tsg_plan_create",
    "tsg_plan_execute", "tsg_plan_execute_stream", "tsg_plan_destroy", "tsg_plan_info",
    "tsg_plan_enqueue", "tsg_plan_sync", "tsg_plan_set_serial", "tsg_plan_describe",
    "tsg_plan_transform", "tsg_plan_free_mode", "tsg_screen_laplace", "tsg_screen_gsylv",
    "tsg_mode_multiply",
    "tsg_residual", "tsg_abi_version",
    "tsg_zlaplace_solve", "tsg_zlaplace_reduced", "tsg_zgsylv_solve", "tsg_zgsylv_reduced",
    "tsg_zmode_multiply", "tsg_zresidual",
    "tsg_slab_bounds", "tsg_slab_pack", "tsg_dplan_create", "tsg_dplan_destroy", "tsg_dplan_info",
    "tsg_dplan_buffers", "tsg_dplan_ipc_export", "tsg_dplan_ipc_import",
    "tsg_dplan_forward_local", "tsg_dplan_forward_split", "tsg_dplan_solve",
    "tsg_dplan_back_local", "tsg_dplan_back_split", "tsg_dplan_status",
]


def _declare(lib: ctypes.CDLL) -> None:
    P = ctypes.c_void_p
    I = ctypes.c_int
    E = ctypes.c_char_p
    sig = {
        "tsg_create": (I, [I, c_int_p, ctypes.POINTER(P)]),
        "tsg_destroy": (None, [P]),
        "tsg_last_error": (E, [P]),
        "tsg_ctx_stream": (P, [P]),
        "tsg_default_opts": (None, [ctypes.POINTER(TsgOpts)]),
        "tsg_abi_version": (I, []),
        "tsg_plan_create": (I, [P, I, I, c_int_p, c_dbl_pp, c_dbl_pp, c_dbl_p, c_dbl_p, I,
                                ctypes.POINTER(TsgOpts), ctypes.POINTER(P)]),
        "tsg_plan_execute": (I, [P, P, P, I, ctypes.POINTER(TsgReport)]),
        "tsg_plan_execute_stream": (I, [P, I, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(TsgReport)]),
        "tsg_plan_destroy": (None, [P]),
        "tsg_plan_enqueue": (I, [P, P, P]),
        "tsg_plan_sync": (I, [P, ctypes.POINTER(TsgReport)]),
        "tsg_plan_set_serial": (I, [P, I]),
        "tsg_plan_transform": (I, [P, I, P, P, P]),
        "tsg_plan_free_mode": (I, [P]),
        "tsg_screen_laplace": (I, [P, I, c_int_p, c_dbl_pp, ctypes.c_double, c_dbl_p, c_int_p, c_int_p]),
        "tsg_screen_gsylv": (I, [P, I, c_int_p, c_dbl_p, c_dbl_p, c_dbl_pp, ctypes.c_double, c_dbl_p, c_int_p,
                                 c_int_p]),
        "tsg_plan_info": (I, [P, ctypes.POINTER(ctypes.c_int64), c_int_p, c_dbl_p]),
        "tsg_plan_describe": (I, [P, ctypes.c_char_p, I]),
        "tsg_residual": (I, [P, I, I, c_int_p, c_dbl_pp, P, P, P, I, c_dbl_p]),
        "tsg_slab_bounds": (I, [I, c_dbl_p, I, I, c_int_p]),
        "tsg_slab_pack": (I, [P, P, P, ctypes.c_longlong, I, I, c_int_p, I, P]),
        "tsg_dplan_create": (I, [P, I, I, I, I, c_int_p, c_dbl_pp, c_dbl_pp, ctypes.POINTER(TsgOpts),
                                 ctypes.POINTER(P)]),
        "tsg_dplan_destroy": (None, [P]),
        "tsg_dplan_info": (I, [P, c_int_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
        "tsg_dplan_buffers": (I, [P, ctypes.POINTER(P), ctypes.POINTER(P)]),
        "tsg_dplan_ipc_export": (I, [P, P]),
        "tsg_dplan_ipc_import": (I, [P, P]),
        "tsg_dplan_forward_local": (I, [P, P, P]),
        "tsg_dplan_forward_split": (I, [P, P]),
        "tsg_dplan_solve": (I, [P, P]),
        "tsg_dplan_back_local": (I, [P, P]),
        "tsg_dplan_back_split": (I, [P, P, P]),
        "tsg_dplan_status": (I, [P, P]),
        "tsylv_solve_laplace": (I, [I, c_int_p, c_dbl_pp, c_dbl_p, I, I, I, c_dbl_p, c_dbl_p, E, I]),
        "tsylv_solve_gsylv": (I, [I, c_int_p, c_dbl_pp, c_dbl_p, c_dbl_p, I, I, I, c_dbl_p,
                                  c_dbl_p, E, I]),
        "tsylv_laplace_recursive": (I, [I, c_int_p, c_dbl_pp, c_dbl_p, I, c_dbl_p, E, I]),
        "tsylv_gsylv_recursive": (I, [I, c_int_p, c_dbl_pp, c_dbl_p, c_dbl_p, I, c_dbl_p, E, I]),
        "tsylv_laplace_merged": (I, [I, c_int_p, c_dbl_pp, c_dbl_p, I, c_dbl_p, E, I]),
        "tsylv_gsylv_merged": (I, [I, c_int_p, c_dbl_pp, c_dbl_p, c_dbl_p, I, c_dbl_p, E, I]),
        "tsylv_solve_sylvester_tri": (I, [I, I, c_dbl_p, c_dbl_p, c_dbl_p, I, c_dbl_p, E, I]),
        "tsylv_solve_gsylv_tri": (I, [I, I, c_dbl_p, c_dbl_p, c_dbl_p, c_dbl_p, I, c_dbl_p, E, I]),
        "tsylv_oracle_solve_laplace": (I, [I, c_int_p, c_dbl_pp, c_dbl_p, c_dbl_p, E, I]),
        "tsylv_oracle_solve_gsylv": (I, [I, c_int_p, c_dbl_pp, c_dbl_p, c_dbl_p, c_dbl_p, E, I]),
        "tsylv_mode_multiply": (I, [I, c_int_p, c_dbl_p, I, c_dbl_p, I, c_dbl_p, E, I]),
        "tsylv_schur": (I, [I, c_dbl_p, c_dbl_p, c_dbl_p, E, I]),
        "tsylv_qz": (I, [I, c_dbl_p, c_dbl_p, c_dbl_p, c_dbl_p, c_dbl_p, c_dbl_p, E, I]),
        "tsylv_residual_laplace": (ctypes.c_double, [I, c_int_p, c_dbl_pp, c_dbl_p, c_dbl_p]),
        "tsylv_residual_gsylv": (ctypes.c_double, [I, c_int_p, c_dbl_pp, c_dbl_p, c_dbl_p, c_dbl_p]),
        "tsylv_check_solvable_laplace": (I, [I, c_int_p, c_dbl_pp, ctypes.c_double, c_dbl_p,
                                             c_int_p, c_int_p, E, I]),
        "tsylv_rng_new": (P, [ctypes.c_uint64]),
        "tsylv_rng_free": (None, [P]),
        "tsylv_rng_uniform": (ctypes.c_double, [P]),
        "tsylv_rng_normal": (ctypes.c_double, [P]),
        "tsylv_rng_randn": (None, [P, c_dbl_p, ctypes.c_size_t]),
        "tsylv_make_problem": (I, [I, I, c_int_p, ctypes.c_uint64, c_dbl_p, c_dbl_p, c_dbl_p]),
    }
    # T = Complex facade: the same signatures over interleaved buffers
    for name in ["solve_laplace", "solve_gsylv", "laplace_recursive", "gsylv_recursive",
                 "laplace_merged", "gsylv_merged", "solve_sylvester_tri", "solve_gsylv_tri",
                 "oracle_solve_laplace", "oracle_solve_gsylv", "mode_multiply", "schur", "qz",
                 "residual_laplace", "residual_gsylv"]:
        sig["tsylv_z" + name] = sig["tsylv_" + name]
    sig["tsylv_zrandom_problem"] = (None, [P, I, I, c_int_p, c_dbl_p, c_dbl_p, c_dbl_p])
    sig["tsg_zlaplace_solve"] = (I, [P, I, c_int_p, c_dbl_pp, c_dbl_pp, P, P,
                                     ctypes.POINTER(TsgOpts), ctypes.POINTER(TsgReport)])
    sig["tsg_zlaplace_reduced"] = (I, [P, I, c_int_p, c_dbl_pp, P, P, ctypes.POINTER(TsgOpts),
                                       ctypes.POINTER(TsgReport)])
    sig["tsg_zgsylv_solve"] = (I, [P, I, c_int_p, P, P, P, P, c_dbl_pp, c_dbl_pp, P, P,
                                   ctypes.POINTER(TsgOpts), ctypes.POINTER(TsgReport)])
    sig["tsg_zgsylv_reduced"] = (I, [P, I, c_int_p, P, P, c_dbl_pp, P, P, ctypes.POINTER(TsgOpts),
                                     ctypes.POINTER(TsgReport)])
    sig["tsg_zmode_multiply"] = (I, [P, I, c_int_p, P, I, P, I, P, ctypes.POINTER(TsgOpts)])
    sig["tsg_zresidual"] = (I, [P, I, I, c_int_p, c_dbl_pp, P, P, P, I, c_dbl_p])
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args


def lib() -> ctypes.CDLL:
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1905_09539_b200.build` "
                "(there is no CPU fallback)")
        _lib = ctypes.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib
