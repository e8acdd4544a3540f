"""TEST INFRASTRUCTURE ONLY.  ctypes binding of oracle/_ref/libtsylv_ref.so,
the reference tsylv solver built from its unmodified headers
(oracle/ref_driver.cpp).  Function names and argument meaning mirror
paper_1905_09539_b200.api so parity tests call both sides identically."""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libtsylv_ref.so")

P = ctypes.c_void_p
I = ctypes.c_int
D = ctypes.c_double
Dp = ctypes.POINTER(ctypes.c_double)
Dpp = ctypes.POINTER(Dp)
Ip = ctypes.POINTER(ctypes.c_int)
E = ctypes.c_char_p

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle`")
        _lib = ctypes.CDLL(LIB_PATH)
        sig = {
            "ref_solve_laplace": (I, [I, Ip, Dpp, Dp, I, I, I, Dp, Dp, E, I]),
            "ref_solve_gsylv": (I, [I, Ip, Dpp, Dp, Dp, I, I, I, Dp, Dp, E, I]),
            "ref_laplace_recursive": (I, [I, Ip, Dpp, Dp, I, Dp, E, I]),
            "ref_gsylv_recursive": (I, [I, Ip, Dpp, Dp, Dp, I, Dp, E, I]),
            "ref_laplace_merged": (I, [I, Ip, Dpp, Dp, I, Dp, E, I]),
            "ref_gsylv_merged": (I, [I, Ip, Dpp, Dp, Dp, I, Dp, E, I]),
            "ref_solve_sylvester_tri": (I, [I, I, Dp, Dp, Dp, I, Dp, E, I]),
            "ref_solve_gsylv_tri": (I, [I, I, Dp, Dp, Dp, Dp, I, Dp, E, I]),
            "ref_baseline_problem": (I, [I, I, Ip, ctypes.c_uint64, Dp, Dp, Dp]),
            "ref_mode_multiply": (I, [I, Ip, Dp, I, Dp, I, Dp, E, I]),
            "ref_schur": (I, [I, Dp, Dp, Dp, E, I]),
            "ref_qz": (I, [I, Dp, Dp, Dp, Dp, Dp, Dp, E, I]),
            "ref_dense_solve_laplace": (I, [I, Ip, Dpp, Dp, Dp, E, I]),
            "ref_dense_solve_gsylv": (I, [I, Ip, Dpp, Dp, Dp, Dp, E, I]),
            "ref_residual_laplace": (D, [I, Ip, Dpp, Dp, Dp]),
            "ref_residual_gsylv": (D, [I, Ip, Dpp, Dp, Dp, Dp]),
            "ref_check_solvable_laplace": (I, [I, Ip, Dpp, D, Dp, Ip, Ip, E, I]),
            "ref_check_solvable_gsylv": (I, [I, Ip, Dpp, Dp, D, Dp, Ip, Ip, E, I]),
            "ref_rng_new": (P, [ctypes.c_uint64]),
            "ref_rng_free": (None, [P]),
            "ref_rng_uniform": (D, [P]),
            "ref_rng_normal": (D, [P]),
            "ref_rng_randn": (None, [P, Dp, ctypes.c_size_t]),
            "ref_random_reduced_laplace": (None, [P, I, Ip, Dp, Dp]),
            "ref_random_laplace_problem": (None, [P, I, Ip, Dp, Dp]),
            "ref_random_reduced_gsylv": (None, [P, I, Ip, Dp, Dp, Dp]),
            "ref_random_gsylv_problem": (None, [P, I, Ip, Dp, Dp, Dp]),
            "ref_randn_quasi_triangular": (None, [P, I, D, D, Dp]),
            # complex scalars (T = Complex), interleaved buffers
            "ref_zsolve_laplace": (I, [I, Ip, Dpp, Dp, I, I, I, Dp, Dp, E, I]),
            "ref_zsolve_gsylv": (I, [I, Ip, Dpp, Dp, Dp, I, I, I, Dp, Dp, E, I]),
            "ref_zlaplace_recursive": (I, [I, Ip, Dpp, Dp, I, Dp, E, I]),
            "ref_zlaplace_merged": (I, [I, Ip, Dpp, Dp, I, Dp, E, I]),
            "ref_zgsylv_recursive": (I, [I, Ip, Dpp, Dp, Dp, I, Dp, E, I]),
            "ref_zgsylv_merged": (I, [I, Ip, Dpp, Dp, Dp, I, Dp, E, I]),
            "ref_zsolve_sylvester_tri": (I, [I, I, Dp, Dp, Dp, I, Dp, E, I]),
            "ref_zsolve_gsylv_tri": (I, [I, I, Dp, Dp, Dp, Dp, I, Dp, E, I]),
            "ref_zmode_multiply": (I, [I, Ip, Dp, I, Dp, I, Dp, E, I]),
            "ref_zschur": (I, [I, Dp, Dp, Dp, E, I]),
            "ref_zqz": (I, [I, Dp, Dp, Dp, Dp, Dp, Dp, E, I]),
            "ref_zdense_solve_laplace": (I, [I, Ip, Dpp, Dp, Dp, E, I]),
            "ref_zdense_solve_gsylv": (I, [I, Ip, Dpp, Dp, Dp, Dp, E, I]),
            "ref_zresidual_laplace": (D, [I, Ip, Dpp, Dp, Dp]),
            "ref_zresidual_gsylv": (D, [I, Ip, Dpp, Dp, Dp, Dp]),
            "ref_zcheck_solvable_laplace": (I, [I, Ip, Dpp, D, Dp, Ip, Ip, E, I]),
            "ref_zcheck_solvable_gsylv": (I, [I, Ip, Dpp, Dp, D, Dp, Ip, Ip, E, I]),
            "ref_zrandn": (None, [P, Dp, ctypes.c_size_t]),
            "ref_run_verify": (I, [ctypes.c_uint64, I, E, D, Dp, E, I]),
            "ref_zrandom_reduced_laplace": (None, [P, I, Ip, Dp, Dp]),
            "ref_zrandom_laplace_problem": (None, [P, I, Ip, Dp, Dp]),
            "ref_zrandom_reduced_gsylv": (None, [P, I, Ip, Dp, Dp, Dp]),
            "ref_zrandom_gsylv_problem": (None, [P, I, Ip, Dp, Dp, Dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data_as(Dp)


def _pp(mats):
    arr = (Dp * len(mats))(*[_p(m) for m in mats])
    return ctypes.cast(arr, Dpp), arr


def _dims(shape):
    return (ctypes.c_int * len(shape))(*shape)


def _chk(rc, err):
    if rc != 0:
        raise RefError(rc, err.value.decode(errors="replace"))


def solve_laplace(coeffs, rhs, strategy=1, arithmetic=0, n_min=0):
    """Returns (X, info[6]) with info = residual, discarded_imag, reduction_s,
    recursion_s, back_transform_s, n_min (laplace.hpp:324-344)."""
    coeffs = [_f(a) for a in coeffs]
    rhs = _f(rhs)
    x = np.zeros(rhs.shape, order="F")
    info = (ctypes.c_double * 6)()
    pp, keep = _pp(coeffs)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_solve_laplace(rhs.ndim, _dims(rhs.shape), pp, _p(rhs), strategy, arithmetic,
                                 n_min, _p(x), info, err, 1024), err)
    return x, list(info)


def solve_gsylv(coeffs, c, rhs, strategy=1, arithmetic=0, n_min=0):
    coeffs = [_f(a) for a in coeffs]
    c = _f(c)
    rhs = _f(rhs)
    x = np.zeros(rhs.shape, order="F")
    info = (ctypes.c_double * 6)()
    pp, keep = _pp(coeffs)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_solve_gsylv(rhs.ndim, _dims(rhs.shape), pp, _p(c), _p(rhs), strategy,
                               arithmetic, n_min, _p(x), info, err, 1024), err)
    return x, list(info)


def laplace_recursive(t, bt, n_min):
    t = [_f(a) for a in t]
    bt = _f(bt)
    x = np.zeros(bt.shape, order="F")
    pp, keep = _pp(t)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_laplace_recursive(bt.ndim, _dims(bt.shape), pp, _p(bt), n_min, _p(x), err,
                                     1024), err)
    return x


def gsylv_recursive(t, tc, bt, n_min):
    t = [_f(a) for a in t]
    tc = _f(tc)
    bt = _f(bt)
    x = np.zeros(bt.shape, order="F")
    pp, keep = _pp(t)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_gsylv_recursive(bt.ndim, _dims(bt.shape), pp, _p(tc), _p(bt), n_min, _p(x),
                                   err, 1024), err)
    return x


def laplace_merged(t, bt, n_min):
    """laplace_merged<double> (laplace.hpp:202-244)."""
    t = [_f(a) for a in t]
    bt = _f(bt)
    x = np.zeros(bt.shape, order="F")
    pp, keep = _pp(t)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_laplace_merged(bt.ndim, _dims(bt.shape), pp, _p(bt), n_min, _p(x), err, 1024),
         err)
    return x


def gsylv_merged(t, tc, bt, n_min):
    """gsylv_merged<double> (gsylv.hpp:167-232)."""
    t = [_f(a) for a in t]
    tc = _f(tc)
    bt = _f(bt)
    x = np.zeros(bt.shape, order="F")
    pp, keep = _pp(t)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_gsylv_merged(bt.ndim, _dims(bt.shape), pp, _p(tc), _p(bt), n_min, _p(x), err,
                                1024), err)
    return x


def solve_sylvester_tri(a1, a2, b, n_min=32):
    """solve_sylvester_tri<double> (sylvester.hpp:194-215): A1 X + X A2^H = B."""
    a1, a2, b = _f(a1), _f(a2), _f(b)
    x = np.zeros(b.shape, order="F")
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_solve_sylvester_tri(a1.shape[0], a2.shape[0], _p(a1), _p(a2), _p(b), n_min,
                                       _p(x), err, 1024), err)
    return x


def solve_gsylv_tri(a1, c, a2, b, n_min=32):
    """solve_gsylv_tri<double> (sylvester.hpp:219-241): A1 X + C X A2^H = B."""
    a1, c, a2, b = _f(a1), _f(c), _f(a2), _f(b)
    x = np.zeros(b.shape, order="F")
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_solve_gsylv_tri(a1.shape[0], a2.shape[0], _p(a1), _p(c), _p(a2), _p(b), n_min,
                                   _p(x), err, 1024), err)
    return x


def baseline_problem(kind, dims, seed=1):
    """BASELINE.json inputs drawn from the reference's RandomStream
    (random.hpp:19-77): returns (coeffs, c or None, rhs).  kind 1 C1,
    2 C2-C4, 5 C5 (coeffs {A, C^T, ..}, c = B)."""
    dims = [int(n) for n in dims]
    co = np.zeros(sum(n * n for n in dims))
    c = np.zeros(dims[0] ** 2)
    rhs = np.zeros(int(np.prod(dims)))
    rc = lib().ref_baseline_problem(kind, len(dims), _dims(dims), seed, _p(co), _p(c), _p(rhs))
    if rc != 0:
        raise RefError(1, f"baseline_problem: bad kind {kind}")
    mats, o = [], 0
    for n in dims:
        mats.append(co[o:o + n * n].reshape((n, n), order="F").copy(order="F"))
        o += n * n
    return (mats, c.reshape((dims[0],) * 2, order="F").copy(order="F") if kind == 5 else None,
            rhs.reshape(dims, order="F"))


def mode_multiply(x, a, mode):
    x = _f(x)
    a = _f(a)
    shape = list(x.shape)
    shape[mode] = a.shape[0]
    y = np.zeros(shape, order="F")
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_mode_multiply(x.ndim, _dims(x.shape), _p(x), a.shape[0], _p(a), mode, _p(y),
                                 err, 1024), err)
    return y


def schur(a):
    a = _f(a)
    n = a.shape[0]
    u = np.zeros((n, n), order="F")
    t = np.zeros((n, n), order="F")
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_schur(n, _p(a), _p(u), _p(t), err, 1024), err)
    return u, t


def qz(a, c):
    a = _f(a)
    c = _f(c)
    n = a.shape[0]
    q, z, s, t = (np.zeros((n, n), order="F") for _ in range(4))
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_qz(n, _p(a), _p(c), _p(q), _p(z), _p(s), _p(t), err, 1024), err)
    return q, z, s, t


def dense_solve_laplace(coeffs, rhs):
    coeffs = [_f(a) for a in coeffs]
    rhs = _f(rhs)
    x = np.zeros(rhs.shape, order="F")
    pp, keep = _pp(coeffs)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_dense_solve_laplace(rhs.ndim, _dims(rhs.shape), pp, _p(rhs), _p(x), err, 1024),
         err)
    return x


def dense_solve_gsylv(coeffs, c, rhs):
    coeffs = [_f(a) for a in coeffs]
    c = _f(c)
    rhs = _f(rhs)
    x = np.zeros(rhs.shape, order="F")
    pp, keep = _pp(coeffs)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_dense_solve_gsylv(rhs.ndim, _dims(rhs.shape), pp, _p(c), _p(rhs), _p(x), err,
                                     1024), err)
    return x


def residual_laplace(coeffs, rhs, x):
    coeffs = [_f(a) for a in coeffs]
    rhs = _f(rhs)
    pp, keep = _pp(coeffs)
    return lib().ref_residual_laplace(rhs.ndim, _dims(rhs.shape), pp, _p(rhs), _p(_f(x)))


def residual_gsylv(coeffs, c, rhs, x):
    coeffs = [_f(a) for a in coeffs]
    rhs = _f(rhs)
    pp, keep = _pp(coeffs)
    return lib().ref_residual_gsylv(rhs.ndim, _dims(rhs.shape), pp, _p(_f(c)), _p(rhs), _p(_f(x)))


class RandomStream:
    def __init__(self, seed):
        self.h = lib().ref_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_rng_free(self.h)
            self.h = None

    def uniform(self):
        return lib().ref_rng_uniform(self.h)

    def normal(self):
        return lib().ref_rng_normal(self.h)

    def randn(self, n):
        out = np.empty(n)
        lib().ref_rng_randn(self.h, _p(out), n)
        return out

    def _unpack(self, dims, flat):
        mats, o = [], 0
        for n in dims:
            mats.append(flat[o:o + n * n].reshape((n, n), order="F").copy(order="F"))
            o += n * n
        return mats

    def reduced_laplace(self, dims):
        """random_reduced_laplace<double> (random.hpp:195-204)."""
        co = np.zeros(sum(n * n for n in dims))
        rhs = np.zeros(int(np.prod(dims)))
        lib().ref_random_reduced_laplace(self.h, len(dims), _dims(dims), _p(co), _p(rhs))
        return self._unpack(dims, co), rhs.reshape(dims, order="F")

    def laplace_problem(self, dims):
        """random_laplace_problem<double> (random.hpp:150-163)."""
        co = np.zeros(sum(n * n for n in dims))
        rhs = np.zeros(int(np.prod(dims)))
        lib().ref_random_laplace_problem(self.h, len(dims), _dims(dims), _p(co), _p(rhs))
        return self._unpack(dims, co), rhs.reshape(dims, order="F")

    def reduced_gsylv(self, dims):
        """random_reduced_gsylv<double> (random.hpp:208-221)."""
        co = np.zeros(sum(n * n for n in dims))
        c = np.zeros(dims[0] ** 2)
        rhs = np.zeros(int(np.prod(dims)))
        lib().ref_random_reduced_gsylv(self.h, len(dims), _dims(dims), _p(co), _p(c), _p(rhs))
        return (self._unpack(dims, co), c.reshape((dims[0],) * 2, order="F"),
                rhs.reshape(dims, order="F"))

    def gsylv_problem(self, dims):
        """random_gsylv_problem<double> (random.hpp:167-189)."""
        co = np.zeros(sum(n * n for n in dims))
        c = np.zeros(dims[0] ** 2)
        rhs = np.zeros(int(np.prod(dims)))
        lib().ref_random_gsylv_problem(self.h, len(dims), _dims(dims), _p(co), _p(c), _p(rhs))
        return (self._unpack(dims, co), c.reshape((dims[0],) * 2, order="F"),
                rhs.reshape(dims, order="F"))

    def quasi_triangular(self, n, diag_shift=0.0, pair_prob=0.5):
        """randn_quasi_triangular (random.hpp:117-146)."""
        out = np.zeros(n * n)
        lib().ref_randn_quasi_triangular(self.h, n, diag_shift, pair_prob, _p(out))
        return out.reshape((n, n), order="F").copy(order="F")


def check_solvable_laplace(t, tol=0.0):
    """The reference's check_solvable_laplace (laplace.hpp:28-43) on reduced
    coefficients: (min_abs, witness, solvable)."""
    t = [_f(m) for m in t]
    pp, keep = _pp(t)
    mn, ok = ctypes.c_double(), ctypes.c_int()
    wit = (ctypes.c_int * len(t))()
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_check_solvable_laplace(len(t), _dims([m.shape[0] for m in t]), pp, tol, ctypes.byref(mn),
                                          wit, ctypes.byref(ok), err, 1024), err)
    return mn.value, list(wit), bool(ok.value)


def check_solvable_gsylv(t, c, tol=0.0):
    """The reference's check_solvable_gsylv (gsylv.hpp:31-50): t = [S, tails..],
    c = the upper triangular pencil partner: (min_abs, witness, solvable)."""
    t = [_f(m) for m in t]
    pp, keep = _pp(t)
    mn, ok = ctypes.c_double(), ctypes.c_int()
    wit = (ctypes.c_int * len(t))()
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_check_solvable_gsylv(len(t), _dims([m.shape[0] for m in t]), pp, _p(_f(c)), tol,
                                        ctypes.byref(mn), wit, ctypes.byref(ok), err, 1024), err)
    return mn.value, list(wit), bool(ok.value)


# ---- complex scalars (T = Complex) ------------------------------------------
# The same reference entry points instantiated for std::complex<double>
# (oracle/ref_driver.cpp ref_z*); numpy complex128 arrays in Fortran order are
# the interleaved layout of std::complex<double>.

def _z(a):
    return np.asfortranarray(np.asarray(a, dtype=np.complex128))


def _zout(shape):
    return np.zeros(shape, dtype=np.complex128, order="F")


def zsolve_laplace(coeffs, rhs, strategy=1, arithmetic=0, n_min=0):
    """solve_laplace<Complex> (laplace.hpp:324-344): (X, info[6])."""
    coeffs = [_z(a) for a in coeffs]
    rhs = _z(rhs)
    x = _zout(rhs.shape)
    info = (ctypes.c_double * 6)()
    pp, keep = _pp(coeffs)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zsolve_laplace(rhs.ndim, _dims(rhs.shape), pp, _p(rhs), strategy, arithmetic,
                                  n_min, _p(x), info, err, 1024), err)
    return x, list(info)


def zsolve_gsylv(coeffs, c, rhs, strategy=1, arithmetic=0, n_min=0):
    """solve_gsylv<Complex> (gsylv.hpp:311-331): (X, info[6])."""
    coeffs = [_z(a) for a in coeffs]
    c, rhs = _z(c), _z(rhs)
    x = _zout(rhs.shape)
    info = (ctypes.c_double * 6)()
    pp, keep = _pp(coeffs)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zsolve_gsylv(rhs.ndim, _dims(rhs.shape), pp, _p(c), _p(rhs), strategy,
                                arithmetic, n_min, _p(x), info, err, 1024), err)
    return x, list(info)


def _zred(fn, t, bt, n_min, tc=None):
    t = [_z(a) for a in t]
    bt = _z(bt)
    x = _zout(bt.shape)
    pp, keep = _pp(t)
    err = ctypes.create_string_buffer(1024)
    if tc is None:
        rc = fn(bt.ndim, _dims(bt.shape), pp, _p(bt), n_min, _p(x), err, 1024)
    else:
        tc = _z(tc)
        rc = fn(bt.ndim, _dims(bt.shape), pp, _p(tc), _p(bt), n_min, _p(x), err, 1024)
    _chk(rc, err)
    return x


def zlaplace_recursive(t, bt, n_min):
    return _zred(lib().ref_zlaplace_recursive, t, bt, n_min)


def zlaplace_merged(t, bt, n_min):
    return _zred(lib().ref_zlaplace_merged, t, bt, n_min)


def zgsylv_recursive(t, tc, bt, n_min):
    return _zred(lib().ref_zgsylv_recursive, t, bt, n_min, tc)


def zgsylv_merged(t, tc, bt, n_min):
    return _zred(lib().ref_zgsylv_merged, t, bt, n_min, tc)


def zsolve_sylvester_tri(a1, a2, b, n_min=32):
    a1, a2, b = _z(a1), _z(a2), _z(b)
    x = _zout(b.shape)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zsolve_sylvester_tri(a1.shape[0], a2.shape[0], _p(a1), _p(a2), _p(b), n_min,
                                        _p(x), err, 1024), err)
    return x


def zsolve_gsylv_tri(a1, c, a2, b, n_min=32):
    a1, c, a2, b = _z(a1), _z(c), _z(a2), _z(b)
    x = _zout(b.shape)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zsolve_gsylv_tri(a1.shape[0], a2.shape[0], _p(a1), _p(c), _p(a2), _p(b),
                                    n_min, _p(x), err, 1024), err)
    return x


def zmode_multiply(x, a, mode):
    x, a = _z(x), _z(a)
    shape = list(x.shape)
    shape[mode] = a.shape[0]
    y = _zout(shape)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zmode_multiply(x.ndim, _dims(x.shape), _p(x), a.shape[0], _p(a), mode, _p(y),
                                  err, 1024), err)
    return y


def zschur(a):
    a = _z(a)
    n = a.shape[0]
    u, t = _zout((n, n)), _zout((n, n))
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zschur(n, _p(a), _p(u), _p(t), err, 1024), err)
    return u, t


def zqz(a, c):
    a, c = _z(a), _z(c)
    n = a.shape[0]
    q, z, s, t = (_zout((n, n)) for _ in range(4))
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zqz(n, _p(a), _p(c), _p(q), _p(z), _p(s), _p(t), err, 1024), err)
    return q, z, s, t


def zdense_solve_laplace(coeffs, rhs):
    coeffs = [_z(a) for a in coeffs]
    rhs = _z(rhs)
    x = _zout(rhs.shape)
    pp, keep = _pp(coeffs)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zdense_solve_laplace(rhs.ndim, _dims(rhs.shape), pp, _p(rhs), _p(x), err,
                                        1024), err)
    return x


def zdense_solve_gsylv(coeffs, c, rhs):
    coeffs = [_z(a) for a in coeffs]
    c, rhs = _z(c), _z(rhs)
    x = _zout(rhs.shape)
    pp, keep = _pp(coeffs)
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zdense_solve_gsylv(rhs.ndim, _dims(rhs.shape), pp, _p(c), _p(rhs), _p(x), err,
                                      1024), err)
    return x


def zresidual_laplace(coeffs, rhs, x):
    coeffs = [_z(a) for a in coeffs]
    rhs = _z(rhs)
    pp, keep = _pp(coeffs)
    return lib().ref_zresidual_laplace(rhs.ndim, _dims(rhs.shape), pp, _p(rhs), _p(_z(x)))


def zresidual_gsylv(coeffs, c, rhs, x):
    coeffs = [_z(a) for a in coeffs]
    rhs = _z(rhs)
    pp, keep = _pp(coeffs)
    return lib().ref_zresidual_gsylv(rhs.ndim, _dims(rhs.shape), pp, _p(_z(c)), _p(rhs),
                                     _p(_z(x)))


def zcheck_solvable_laplace(t, tol=0.0):
    t = [_z(m) for m in t]
    pp, keep = _pp(t)
    mn, ok = ctypes.c_double(), ctypes.c_int()
    wit = (ctypes.c_int * len(t))()
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zcheck_solvable_laplace(len(t), _dims([m.shape[0] for m in t]), pp, tol,
                                           ctypes.byref(mn), wit, ctypes.byref(ok), err, 1024), err)
    return mn.value, list(wit), bool(ok.value)


def zcheck_solvable_gsylv(t, c, tol=0.0):
    t = [_z(m) for m in t]
    pp, keep = _pp(t)
    mn, ok = ctypes.c_double(), ctypes.c_int()
    wit = (ctypes.c_int * len(t))()
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_zcheck_solvable_gsylv(len(t), _dims([m.shape[0] for m in t]), pp, _p(_z(c)),
                                         tol, ctypes.byref(mn), wit, ctypes.byref(ok), err, 1024),
         err)
    return mn.value, list(wit), bool(ok.value)


class ZRandomStream(RandomStream):
    """The reference RandomStream drawing T = Complex instances
    (random.hpp:64-223 with is_complex_v<T>)."""

    def _zunpack(self, dims, flat):
        mats, o = [], 0
        for n in dims:
            mats.append(flat[o:o + n * n].reshape((n, n), order="F").copy(order="F"))
            o += n * n
        return mats

    def zrandn(self, n):
        out = np.zeros(n, dtype=np.complex128)
        lib().ref_zrandn(self.h, _p(out), n)
        return out

    def _draw(self, fn, dims, with_c):
        co = np.zeros(sum(n * n for n in dims), dtype=np.complex128)
        c = np.zeros(dims[0] ** 2, dtype=np.complex128)
        rhs = np.zeros(int(np.prod(dims)), dtype=np.complex128)
        if with_c:
            fn(self.h, len(dims), _dims(dims), _p(co), _p(c), _p(rhs))
            return (self._zunpack(dims, co), c.reshape((dims[0],) * 2, order="F"),
                    rhs.reshape(dims, order="F"))
        fn(self.h, len(dims), _dims(dims), _p(co), _p(rhs))
        return self._zunpack(dims, co), rhs.reshape(dims, order="F")

    def reduced_laplace(self, dims):
        return self._draw(lib().ref_zrandom_reduced_laplace, dims, False)

    def laplace_problem(self, dims):
        return self._draw(lib().ref_zrandom_laplace_problem, dims, False)

    def reduced_gsylv(self, dims):
        return self._draw(lib().ref_zrandom_reduced_gsylv, dims, True)

    def gsylv_problem(self, dims):
        return self._draw(lib().ref_zrandom_gsylv_problem, dims, True)


def run_verify(seed, per_family=50, out_dir="", tol=1e-9):
    """The reference's run_verify (bench.hpp:255-352), writing its
    verify_<family>_<k>.json files to out_dir when given."""
    out = (ctypes.c_double * 4)()
    err = ctypes.create_string_buffer(1024)
    _chk(lib().ref_run_verify(seed, per_family, out_dir.encode(), tol, out, err, 1024), err)
    return {"pass": bool(out[0]), "instances": int(out[1]), "worst_rel": out[2],
            "worst_residual": out[3]}
