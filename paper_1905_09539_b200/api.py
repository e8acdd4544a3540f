"""Python host mirror of the reference tsylv API (proj/include/tsylv).

Same names, argument meaning and error behaviour as the reference's C++ entry
points; every call goes to the C++ drop-in facade inside ``libtsylv_gpu.so``
(no CPU fallback).  Tensors are numpy arrays in Fortran order (mode 0 fastest,
the reference layout, tensor.hpp:19-27); matrices are (n, n) float64 arrays.

    solve_laplace(p, cfg)          laplace.hpp:324-344
    solve_gsylv(p, cfg)            gsylv.hpp:311-331
    laplace_recursive(T, Bt, nmin) laplace.hpp:185-195
    gsylv_recursive(T, C, Bt, nmin) gsylv.hpp:149-159
    laplace_merged(T, Bt, nmin)    laplace.hpp:202-244
    gsylv_merged(T, C, Bt, nmin)   gsylv.hpp:167-232
    solve_sylvester_tri(A1, A2, B, nmin)     sylvester.hpp:194-215
    solve_gsylv_tri(A1, C, A2, B, nmin)      sylvester.hpp:219-241
    oracle.residual(p, X), oracle.solve(p)   oracle.hpp:205-268
    mode_multiply(X, A, mode)      tensor.hpp:187-231
    schur(A), qz(A, C)             kernels.hpp:78-156 (host LAPACK, shared setup)

Complex problems (T = Complex): pass complex128 arrays
to the same functions; they dispatch to the tsylv_z* facade (complex Schur /
QZ on the host, complex DMMA transforms and the eigen-decoupled triangular
solve on the GPU).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from ._lib import TsgOpts, TsgReport, c_dbl_p, c_dbl_pp, c_int_p, lib


# ---- errors (errors.hpp:13-62) ---------------------------------------------
class dimension_error(ValueError):
    pass


class singular_error(RuntimeError):
    pass


class factorization_error(RuntimeError):
    pass


class gpu_error(RuntimeError):
    pass


def _raise(rc: int, err: ctypes.Array) -> None:
    if rc == 0:
        return
    msg = err.value.decode(errors="replace")
    if rc == 1:
        raise dimension_error(msg)
    if rc == 2:
        raise singular_error(msg)
    if rc == 3:
        raise factorization_error(msg)
    if rc == 4:
        raise ValueError(msg)  # std::invalid_argument
    raise gpu_error(msg)


# ---- config (config.hpp:11-68) -----------------------------------------------
class Strategy(enum.IntEnum):
    recursion_only = 0
    merge = 1


class Arithmetic(enum.IntEnum):
    complex_triangular = 0
    real_quasitriangular = 1


@dataclass
class SolverConfig:
    n_min: int = 0
    strategy: Strategy = Strategy.merge
    arithmetic: Arithmetic = Arithmetic.complex_triangular


@dataclass
class PhaseTimings:
    reduction_s: float = 0.0
    recursion_s: float = 0.0
    back_transform_s: float = 0.0


@dataclass
class SolveReport:
    solution: np.ndarray
    residual: float
    discarded_imag: float
    timings: PhaseTimings
    n_min: int
    strategy: Strategy
    gpu: dict = field(default_factory=dict)


@dataclass
class LaplaceProblem:
    coeffs: list
    rhs: np.ndarray

    def order(self) -> int:
        return len(self.coeffs)

    def dims(self) -> list:
        return [int(a.shape[0]) for a in self.coeffs]


@dataclass
class GSylvProblem:
    coeffs: list
    c: np.ndarray
    rhs: np.ndarray

    def order(self) -> int:
        return len(self.coeffs)

    def dims(self) -> list:
        return [int(a.shape[0]) for a in self.coeffs]


# ---- marshalling helpers -------------------------------------------------------
def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _z(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.complex128))


def _cplx(*arrays) -> bool:
    """T = Complex when any input is complex: the
    tsylv_z* entry points take interleaved std::complex<double> buffers,
    which is the memory layout of numpy complex128."""
    for a in arrays:
        if isinstance(a, (list, tuple)):
            if any(np.iscomplexobj(v) for v in a):
                return True
        elif np.iscomplexobj(a):
            return True
    return False


def _conv(z: bool):
    return _z if z else _f


def _zeros(shape, z: bool) -> np.ndarray:
    return np.zeros(shape, dtype=np.complex128 if z else np.float64, order="F")


def _fn(name: str, z: bool):
    return getattr(lib(), name.replace("tsylv_", "tsylv_z", 1) if z else name)


def _dims(rhs: np.ndarray) -> ctypes.Array:
    return (ctypes.c_int * rhs.ndim)(*rhs.shape)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(c_dbl_p)


def _ptrs(mats: list):
    arr = (c_dbl_p * len(mats))(*[_ptr(m) for m in mats])
    return ctypes.cast(arr, c_dbl_pp), arr


def _err():
    return ctypes.create_string_buffer(1024)


def _check_problem(coeffs, rhs, who):
    if len(coeffs) < 2:
        raise dimension_error(f"{who}: need order d >= 2")
    if rhs.ndim != len(coeffs):
        raise dimension_error(f"{who}: rhs order does not match coefficient count")
    for m, a in enumerate(coeffs):
        if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] == 0:
            raise dimension_error(f"{who}: coefficient {m} must be square, non-empty")
        if a.shape[0] != rhs.shape[m]:
            raise dimension_error(f"{who}: coefficient {m} does not match rhs extent")


def _report(x, info, cfg) -> SolveReport:
    return SolveReport(
        solution=x, residual=info[0], discarded_imag=info[1],
        timings=PhaseTimings(info[2], info[3], info[4]), n_min=int(info[5]),
        strategy=Strategy(int(cfg.strategy)),
        gpu=dict(fwd_ms=info[6], solve_ms=info[7], back_ms=info[8], h2d_ms=info[9],
                 d2h_ms=info[10], total_ms=info[11], flops_alg=info[12], flops_exec=info[13]))


# ---- entry points ------------------------------------------------------------------
def solve_laplace(p: LaplaceProblem, cfg: SolverConfig | None = None) -> SolveReport:
    cfg = cfg or SolverConfig()
    z = _cplx(p.coeffs, p.rhs)
    cv = _conv(z)
    coeffs = [cv(a) for a in p.coeffs]
    rhs = cv(p.rhs)
    _check_problem(coeffs, rhs, "LaplaceProblem")
    x = _zeros(rhs.shape, z)
    info = (ctypes.c_double * 14)()
    pp, keep = _ptrs(coeffs)
    err = _err()
    rc = _fn("tsylv_solve_laplace", z)(rhs.ndim, _dims(rhs), pp, _ptr(rhs), int(cfg.strategy),
                                   int(cfg.arithmetic), int(cfg.n_min), _ptr(x), info, err, 1024)
    _raise(rc, err)
    return _report(x, list(info), cfg)


def solve_gsylv(p: GSylvProblem, cfg: SolverConfig | None = None) -> SolveReport:
    cfg = cfg or SolverConfig()
    z = _cplx(p.coeffs, p.c, p.rhs)
    cv = _conv(z)
    coeffs = [cv(a) for a in p.coeffs]
    c = cv(p.c)
    rhs = cv(p.rhs)
    _check_problem(coeffs, rhs, "GSylvProblem")
    if c.shape != coeffs[0].shape:
        raise dimension_error("GSylvProblem: C must be square with the order of A_0")
    x = _zeros(rhs.shape, z)
    info = (ctypes.c_double * 14)()
    pp, keep = _ptrs(coeffs)
    err = _err()
    rc = _fn("tsylv_solve_gsylv", z)(rhs.ndim, _dims(rhs), pp, _ptr(c), _ptr(rhs), int(cfg.strategy),
                                 int(cfg.arithmetic), int(cfg.n_min), _ptr(x), info, err, 1024)
    _raise(rc, err)
    return _report(x, list(info), cfg)


def laplace_recursive(coeffs: list, b: np.ndarray, n_min: int) -> np.ndarray:
    z = _cplx(coeffs, b)
    cv = _conv(z)
    coeffs = [cv(a) for a in coeffs]
    b = cv(b)
    if b.ndim != len(coeffs):
        raise dimension_error("laplace_recursive: rhs order does not match coefficient count")
    x = _zeros(b.shape, z)
    pp, keep = _ptrs(coeffs)
    err = _err()
    rc = _fn("tsylv_laplace_recursive", z)(b.ndim, _dims(b), pp, _ptr(b), int(n_min), _ptr(x), err, 1024)
    _raise(rc, err)
    return x


def gsylv_recursive(coeffs: list, c: np.ndarray, b: np.ndarray, n_min: int) -> np.ndarray:
    z = _cplx(coeffs, c, b)
    cv = _conv(z)
    coeffs = [cv(a) for a in coeffs]
    c = cv(c)
    b = cv(b)
    if b.ndim != len(coeffs):
        raise dimension_error("gsylv_recursive: rhs order does not match coefficient count")
    x = _zeros(b.shape, z)
    pp, keep = _ptrs(coeffs)
    err = _err()
    rc = _fn("tsylv_gsylv_recursive", z)(b.ndim, _dims(b), pp, _ptr(c), _ptr(b), int(n_min), _ptr(x),
                                     err, 1024)
    _raise(rc, err)
    return x


def laplace_merged(coeffs: list, b: np.ndarray, n_min: int) -> np.ndarray:
    z = _cplx(coeffs, b)
    cv = _conv(z)
    coeffs = [cv(a) for a in coeffs]
    b = cv(b)
    if b.ndim != len(coeffs):
        raise dimension_error("laplace_merged: rhs order does not match coefficient count")
    x = _zeros(b.shape, z)
    pp, keep = _ptrs(coeffs)
    err = _err()
    rc = _fn("tsylv_laplace_merged", z)(b.ndim, _dims(b), pp, _ptr(b), int(n_min), _ptr(x), err, 1024)
    _raise(rc, err)
    return x


def gsylv_merged(coeffs: list, c: np.ndarray, b: np.ndarray, n_min: int) -> np.ndarray:
    z = _cplx(coeffs, c, b)
    cv = _conv(z)
    coeffs = [cv(a) for a in coeffs]
    c = cv(c)
    b = cv(b)
    if b.ndim != len(coeffs):
        raise dimension_error("gsylv_merged: rhs order does not match coefficient count")
    x = _zeros(b.shape, z)
    pp, keep = _ptrs(coeffs)
    err = _err()
    rc = _fn("tsylv_gsylv_merged", z)(b.ndim, _dims(b), pp, _ptr(c), _ptr(b), int(n_min), _ptr(x),
                                  err, 1024)
    _raise(rc, err)
    return x


def _mat2(a, who, cv=_f):
    a = cv(a)
    if a.ndim != 2:
        raise dimension_error(f"{who}: expected a matrix")
    return a


def solve_sylvester_tri(a1: np.ndarray, a2: np.ndarray, b: np.ndarray, n_min: int = 32) -> np.ndarray:
    """A1 X + X A2^H = B with (quasi-)triangular A1, A2 (sylvester.hpp:194-215)."""
    z = _cplx(a1, a2, b)
    a1, a2, b = (_mat2(v, "solve_sylvester_tri", _conv(z)) for v in (a1, a2, b))
    if a1.shape[0] != a1.shape[1] or a2.shape[0] != a2.shape[1]:
        raise dimension_error("solve_sylvester_tri: coefficients must be square")
    if b.shape != (a1.shape[0], a2.shape[0]):
        raise dimension_error(f"solve_sylvester_tri: rhs is {b.shape[0]}x{b.shape[1]}, expected "
                              f"{a1.shape[0]}x{a2.shape[0]}")
    x = _zeros(b.shape, z)
    err = _err()
    rc = _fn("tsylv_solve_sylvester_tri", z)(a1.shape[0], a2.shape[0], _ptr(a1), _ptr(a2), _ptr(b),
                                         int(n_min), _ptr(x), err, 1024)
    _raise(rc, err)
    return x


def solve_gsylv_tri(a1: np.ndarray, c: np.ndarray, a2: np.ndarray, b: np.ndarray,
                    n_min: int = 32) -> np.ndarray:
    """A1 X + C X A2^H = B, (A1, C) in generalized Schur form (sylvester.hpp:219-241)."""
    z = _cplx(a1, c, a2, b)
    a1, c, a2, b = (_mat2(v, "solve_gsylv_tri", _conv(z)) for v in (a1, c, a2, b))
    if a1.shape[0] != a1.shape[1] or a2.shape[0] != a2.shape[1]:
        raise dimension_error("solve_gsylv_tri: coefficients must be square")
    if c.shape != a1.shape:
        raise dimension_error("solve_gsylv_tri: C must match A1")
    if b.shape != (a1.shape[0], a2.shape[0]):
        raise dimension_error(f"solve_gsylv_tri: rhs is {b.shape[0]}x{b.shape[1]}, expected "
                              f"{a1.shape[0]}x{a2.shape[0]}")
    x = _zeros(b.shape, z)
    err = _err()
    rc = _fn("tsylv_solve_gsylv_tri", z)(a1.shape[0], a2.shape[0], _ptr(a1), _ptr(c), _ptr(a2), _ptr(b),
                                     int(n_min), _ptr(x), err, 1024)
    _raise(rc, err)
    return x


class oracle:
    """tsylv::oracle (oracle.hpp:205-268): residual on the device, dense
    assemble-and-LU solve (N <= 4096) as the independent cross-check."""

    @staticmethod
    def residual(p, x: np.ndarray) -> float:
        return residual(p, x)

    @staticmethod
    def solve(p) -> np.ndarray:
        z = _cplx(p.coeffs, p.rhs, getattr(p, "c", None))
        cv = _conv(z)
        coeffs = [cv(a) for a in p.coeffs]
        rhs = cv(p.rhs)
        _check_problem(coeffs, rhs, "oracle::solve")
        x = _zeros(rhs.shape, z)
        pp, keep = _ptrs(coeffs)
        err = _err()
        if isinstance(p, GSylvProblem):
            rc = _fn("tsylv_oracle_solve_gsylv", z)(rhs.ndim, _dims(rhs), pp, _ptr(cv(p.c)),
                                                    _ptr(rhs), _ptr(x), err, 1024)
        else:
            rc = _fn("tsylv_oracle_solve_laplace", z)(rhs.ndim, _dims(rhs), pp, _ptr(rhs), _ptr(x),
                                                  err, 1024)
        _raise(rc, err)
        return x


def mode_multiply(x: np.ndarray, a: np.ndarray, mode: int) -> np.ndarray:
    z = _cplx(x, a)
    x = _conv(z)(x)
    a = _conv(z)(a)
    if not 0 <= mode < x.ndim:
        raise dimension_error("mode_multiply: mode out of range")
    shape = list(x.shape)
    shape[mode] = a.shape[0]
    y = _zeros(shape, z)
    err = _err()
    rc = _fn("tsylv_mode_multiply", z)(x.ndim, _dims(x), _ptr(x), int(a.shape[0]), _ptr(a), int(mode),
                                   _ptr(y), err, 1024)
    _raise(rc, err)
    return y


def schur(a: np.ndarray):
    z = _cplx(a)
    a = _conv(z)(a)
    n = a.shape[0]
    u = _zeros((n, n), z)
    t = _zeros((n, n), z)
    err = _err()
    _raise(_fn("tsylv_schur", z)(n, _ptr(a), _ptr(u), _ptr(t), err, 1024), err)
    return u, t


def qz(a: np.ndarray, c: np.ndarray):
    cz = _cplx(a, c)
    a = _conv(cz)(a)
    c = _conv(cz)(c)
    n = a.shape[0]
    q, z, s, t = (_zeros((n, n), cz) for _ in range(4))
    err = _err()
    _raise(_fn("tsylv_qz", cz)(n, _ptr(a), _ptr(c), _ptr(q), _ptr(z), _ptr(s), _ptr(t), err, 1024),
           err)
    return q, z, s, t


def residual(p, x: np.ndarray) -> float:
    z = _cplx(p.coeffs, p.rhs, x, getattr(p, "c", None))
    cv = _conv(z)
    x = cv(x)
    coeffs = [cv(a) for a in p.coeffs]
    rhs = cv(p.rhs)
    pp, keep = _ptrs(coeffs)
    if isinstance(p, GSylvProblem):
        return _fn("tsylv_residual_gsylv", z)(rhs.ndim, _dims(rhs), pp, _ptr(cv(p.c)), _ptr(rhs),
                                             _ptr(x))
    return _fn("tsylv_residual_laplace", z)(rhs.ndim, _dims(rhs), pp, _ptr(rhs), _ptr(x))


class RandomStream:
    """The reference's deterministic stream (random.hpp:19-62), in C++."""

    def __init__(self, seed: int):
        self._h = lib().tsylv_rng_new(seed)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().tsylv_rng_free(self._h)
            self._h = None

    def uniform(self) -> float:
        return lib().tsylv_rng_uniform(self._h)

    def normal(self) -> float:
        return lib().tsylv_rng_normal(self._h)

    def randn(self, n: int) -> np.ndarray:
        out = np.empty(n)
        lib().tsylv_rng_randn(self._h, _ptr(out), n)
        return out


def random_problem(which: str, dims, seed: int = 1, scalar=np.complex128):
    """The reference's correctness-suite instances drawn from its stream
    (random.hpp:150-221) with T = Complex: which = "laplace" (dense,
    random_laplace_problem), "reduced_laplace", "gsylv", "reduced_gsylv"."""
    if scalar is not np.complex128:
        raise ValueError("random_problem: only complex128 (the real configs use make_problem)")
    code = {"laplace": 0, "reduced_laplace": 1, "gsylv": 2, "reduced_gsylv": 3}[which]
    dims = [int(n) for n in dims]
    d = len(dims)
    co = np.zeros(sum(n * n for n in dims), dtype=np.complex128)
    c = np.zeros(dims[0] ** 2, dtype=np.complex128)
    rhs = np.zeros(int(np.prod(dims)), dtype=np.complex128)
    rs = RandomStream(seed)
    lib().tsylv_zrandom_problem(rs._h, code, d, (ctypes.c_int * d)(*dims), _ptr(co), _ptr(c),
                                _ptr(rhs))
    mats, o = [], 0
    for n in dims:
        mats.append(co[o:o + n * n].reshape((n, n), order="F").copy(order="F"))
        o += n * n
    rhs = rhs.reshape(dims, order="F")
    if code >= 2:
        return GSylvProblem(mats, c.reshape((dims[0], dims[0]), order="F").copy(order="F"), rhs)
    return LaplaceProblem(mats, rhs)


def make_problem(kind: int, dims, seed: int = 1):
    """BASELINE.json inputs (include/tsylv/random.hpp): kind 1 convection-
    diffusion Laplace (C1), 2 G/sqrt(n)+3I Laplace (C2-C4), 5 gsylv (C5)."""
    dims = [int(n) for n in dims]
    d = len(dims)
    coeffs = np.zeros(sum(n * n for n in dims))
    c = np.zeros(dims[0] * dims[0])
    rhs = np.zeros(int(np.prod(dims)))
    rc = lib().tsylv_make_problem(kind, d, (ctypes.c_int * d)(*dims), seed, _ptr(coeffs), _ptr(c),
                                  _ptr(rhs))
    if rc != 0:
        raise dimension_error(f"make_problem: bad kind/dims {kind} {dims}")
    mats, o = [], 0
    for n in dims:
        mats.append(coeffs[o:o + n * n].reshape((n, n), order="F").copy(order="F"))
        o += n * n
    rhs = rhs.reshape(dims, order="F")
    if kind == 5:
        return GSylvProblem(mats, c.reshape((dims[0], dims[0]), order="F").copy(order="F"), rhs)
    return LaplaceProblem(mats, rhs)


# ---- solvability screen (reference solvability.hpp:31-116) ----------------
_screen_ctx = None


def _ctx():
    global _screen_ctx
    if _screen_ctx is None:
        from .plan import Context
        _screen_ctx = Context(0)
    return _screen_ctx


def screen_laplace(t: list, tol: float = 0.0):
    """GPU screen of the reduced Laplace operator (quasi-triangular factors):
    (min |eigenvalue|, witness per mode, solvable) — tsg_screen_laplace."""
    t = [_f(m) for m in t]
    d = len(t)
    pp, keep = _ptrs(t)
    mn, ok = ctypes.c_double(), ctypes.c_int()
    wit = (ctypes.c_int * d)()
    ctx = _ctx()
    rc = lib().tsg_screen_laplace(ctx.h, d, (ctypes.c_int * d)(*[m.shape[0] for m in t]), pp, tol,
                                  ctypes.byref(mn), wit, ctypes.byref(ok))
    if rc != 0:
        raise gpu_error(f"tsg_screen_laplace failed ({rc}): {ctx.error()}")
    return mn.value, list(wit), bool(ok.value)


def screen_gsylv(s: np.ndarray, tc: np.ndarray, tails: list, tol: float = 0.0):
    """GPU screen of the reduced gsylv pencil: S, Tc (QZ pair of mode 0) and
    the tail factors — tsg_screen_gsylv."""
    s, tc = _f(s), _f(tc)
    tails = [_f(m) for m in tails]
    d = 1 + len(tails)
    pp, keep = _ptrs(tails)
    mn, ok = ctypes.c_double(), ctypes.c_int()
    wit = (ctypes.c_int * d)()
    dims = [s.shape[0]] + [m.shape[0] for m in tails]
    ctx = _ctx()
    rc = lib().tsg_screen_gsylv(ctx.h, d, (ctypes.c_int * d)(*dims), _ptr(s), _ptr(tc), pp, tol,
                                ctypes.byref(mn), wit, ctypes.byref(ok))
    if rc != 0:
        raise gpu_error(f"tsg_screen_gsylv failed ({rc}): {ctx.error()}")
    return mn.value, list(wit), bool(ok.value)
