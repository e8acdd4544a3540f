"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference tsylv
algorithms for the Schur-basis solve path (checker, never product).

Pinned against the reference's own build (oracle/_ref/libtsylv_ref.so, see
tests/test_oracle_restate.py) and against the committed golden fixtures
(tests/golden/, generated from oracle/_ref by tests/golden/make_golden.py).

Every function cites the reference file:line it restates (paths relative to
/root/reference/proj).  Real arithmetic only (the real quasi-triangular
recursion path, Arithmetic::real_quasitriangular); sizes are meant to be small
(pure-Python recursion).
"""
from __future__ import annotations

import math

import numpy as np

U = np.finfo(np.float64).eps / 2  # unit roundoff, scalar.hpp:20-22


class DimensionError(ValueError):
    pass


class SingularError(RuntimeError):
    pass


# ---- RandomStream (random.hpp:19-62): mt19937_64 + Box-Muller ----------------
class MT19937_64:
    """Restatement of std::mt19937_64 (the C++ standard's published
    parameters: w=64, n=312, m=156, r=31, a=0xB5026F5AA96619E9,
    u=29 d=0x5555555555555555, s=17 b=0x71D67FFFEDA60000,
    t=37 c=0xFFF7EEE000000000, l=43, f=6364136223846793005)."""

    N, M = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
    MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        self.mt = [0] * self.N
        self.mt[0] = seed & self.MASK
        for i in range(1, self.N):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self.MASK
        self.idx = self.N

    def _twist(self):
        mt = self.mt
        for i in range(self.N):
            x = (mt[i] & self.UM) | (mt[(i + 1) % self.N] & self.LM)
            xa = x >> 1
            if x & 1:
                xa ^= self.MATRIX_A
            mt[i] = mt[(i + self.M) % self.N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self.MASK


class RandomStream:
    """random.hpp:19-62: uniform = (eng() >> 11) * 2^-53; Box-Muller normal
    returning r*cos and caching r*sin."""

    def __init__(self, seed: int):
        self.eng = MT19937_64(seed)
        self.spare = None

    def uniform(self) -> float:
        return (self.eng() >> 11) * 2.0 ** -53

    def normal(self) -> float:
        if self.spare is not None:
            v, self.spare = self.spare, None
            return v
        u1 = 1.0 - self.uniform()
        u2 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        th = 2.0 * math.pi * u2
        self.spare = r * math.sin(th)
        return r * math.cos(th)

    def randn(self, n: int) -> np.ndarray:
        return np.array([self.normal() for _ in range(n)])


def randn_matrix(rs: RandomStream, r: int, c: int) -> np.ndarray:
    """random.hpp:64-69 (column-major fill)."""
    return rs.randn(r * c).reshape((r, c), order="F")


def randn_tensor(rs: RandomStream, dims) -> np.ndarray:
    """random.hpp:71-77 (storage order = mode 0 fastest)."""
    return rs.randn(int(np.prod(dims))).reshape(dims, order="F")


def baseline_problem(kind: int, dims, seed: int = 1):
    """BASELINE.json configs (SURVEY §8d synthetic inputs).  kind 1: C1
    convection-diffusion; kind 2: G/sqrt(n)+3I; kind 5: gsylv C5 posed as
    coeffs {A, C^T, ..., C^T}, c = B."""
    rs = RandomStream(seed)
    if kind == 5:
        n0, nc = dims[0], dims[1]
        A = randn_matrix(rs, n0, n0) / math.sqrt(n0) + 4.0 * np.eye(n0)
        B = randn_matrix(rs, n0, n0) / math.sqrt(n0)
        C = randn_matrix(rs, nc, nc) / (2.0 * math.sqrt(nc))
        rhs = randn_tensor(rs, dims)
        return [A] + [C.T.copy()] * (len(dims) - 1), B, rhs
    coeffs = []
    for n in dims:
        if kind == 1:
            c = 0.5 + 1.5 * rs.uniform()
            h2, h1 = (n + 1) ** 2, c * (n + 1) / 2.0
            a = np.zeros((n, n))
            for i in range(n):
                a[i, i] = 2 * h2
                if i + 1 < n:
                    a[i, i + 1] = -h2 + h1
                    a[i + 1, i] = -h2 - h1
            coeffs.append(a)
        else:
            coeffs.append(randn_matrix(rs, n, n) / math.sqrt(n) + 3.0 * np.eye(n))
    return coeffs, None, randn_tensor(rs, dims)


# ---- tensor primitives (tensor.hpp:131-231) --------------------------------------
def mode_multiply(x: np.ndarray, a: np.ndarray, mode: int) -> np.ndarray:
    """Y = X x_mode A, Y_(mode) = A X_(mode) (tensor.hpp:184-231)."""
    if a.shape[1] != x.shape[mode]:
        raise DimensionError("mode_multiply: A columns != mode extent")
    y = np.tensordot(a, x, axes=([1], [mode]))  # new axis first
    return np.asfortranarray(np.moveaxis(y, 0, mode))


# ---- structure (matrix.hpp:152-172, kernels.hpp:288-304) ---------------------------
def is_upper_quasi_triangular(t: np.ndarray) -> bool:
    n = t.shape[0]
    if np.any(np.tril(t, -2) != 0):
        return False
    sub = np.diag(t, -1)
    return not np.any((sub[:-1] != 0) & (sub[1:] != 0))


def split_index(t: np.ndarray, lo: int, hi: int) -> int:
    """sylvester.hpp:43-49: midpoint, bumped past a 2x2 block."""
    k = lo + (hi - lo) // 2
    if t[k, k - 1] != 0:
        k += 1
    return k


def lower_block_partition(t: np.ndarray) -> list:
    """kernels.hpp:266-284: finest block upper triangular partition."""
    n = t.shape[0]
    sizes, reach, start = [], 0, 0
    for j in range(n):
        nz = np.nonzero(t[j + 1:, j])[0]
        if nz.size:
            reach = max(reach, j + 1 + int(nz[-1]))
        if reach <= j:
            sizes.append(j + 1 - start)
            start = j + 1
    return sizes


def block_back_substitution(t: np.ndarray, b: np.ndarray, sizes=None) -> np.ndarray:
    """kernels.hpp:179-261: triangular back-substitution, or block variant
    with a dense partial-pivoting solve per diagonal block; zero pivots
    (<= u*||T||_F) raise SingularError."""
    n = t.shape[0]
    tiny = U * np.linalg.norm(t)
    b = b.astype(np.float64).copy()
    if sizes is None:
        for j in range(n - 1, -1, -1):
            if abs(t[j, j]) <= tiny:
                raise SingularError(f"zero pivot at {j}")
            b[j] /= t[j, j]
            b[:j] -= t[:j, j] * b[j]
        return b
    e = n
    for sz in reversed(sizes):
        s = e - sz
        blk = t[s:e, s:e]
        if np.min(np.abs(np.linalg.svd(blk, compute_uv=False))) <= tiny:
            raise SingularError(f"singular block at [{s},{e})")
        b[s:e] = np.linalg.solve(blk, b[s:e])
        b[:s] -= t[:s, s:e] @ b[s:e]
        e = s
    return b


# ---- Laplace recursion (laplace.hpp:83-195) --------------------------------------------
def _pick_split(a, win, n_min):
    """laplace.hpp:83-96: largest splittable window > n_min, ties -> lowest mode."""
    best, best_size, best_k = -1, n_min, -1
    for m, (lo, hi) in enumerate(win):
        size = hi - lo
        if size <= best_size:
            continue
        k = split_index(a[m], lo, hi)
        if k == hi:
            continue
        best, best_size, best_k = m, size, k
    return best, best_k


def _lap_base(a, win, b, all_tri):
    """laplace.hpp:99-132: assemble the Kronecker-sum block, back-substitute."""
    big = b.size
    op = np.zeros((big, big))
    stride = 1
    for m, (lo, hi) in enumerate(win):
        n = hi - lo
        outer = big // (stride * n)
        blk = a[m][lo:hi, lo:hi]
        for o in range(outer):
            for j in range(n):
                for i in range(min(j + 2, n)):
                    v = blk[i, j]
                    if v == 0:
                        continue
                    rb = o * stride * n + i * stride
                    cb = o * stride * n + j * stride
                    idx = np.arange(stride)
                    op[rb + idx, cb + idx] += v
        stride *= n
    vec = b.reshape(-1, order="F")
    sol = block_back_substitution(op, vec, None if all_tri else lower_block_partition(op))
    return sol.reshape(b.shape, order="F")


def _lap_rec(a, win, b, n_min, all_tri):
    """laplace.hpp:134-153: split, solve trailing block, update, solve head."""
    mu, k = _pick_split(a, win, n_min)
    if mu < 0:
        return _lap_base(a, win, b, all_tri)
    lo, hi = win[mu]
    sl1 = [slice(None)] * b.ndim
    sl2 = [slice(None)] * b.ndim
    sl1[mu] = slice(0, k - lo)
    sl2[mu] = slice(k - lo, None)
    b1, b2 = b[tuple(sl1)].copy(), b[tuple(sl2)].copy()
    w2 = list(win)
    w2[mu] = (k, hi)
    x2 = _lap_rec(a, w2, b2, n_min, all_tri)
    b1 -= mode_multiply(x2, a[mu][lo:k, k:hi], mu)  # laplace.hpp:147
    w1 = list(win)
    w1[mu] = (lo, k)
    x1 = _lap_rec(a, w1, b1, n_min, all_tri)
    return np.concatenate([x1, x2], axis=mu)


def laplace_recursive(t: list, b: np.ndarray, n_min: int) -> np.ndarray:
    """laplace.hpp:185-195 (require_reduced :155-178)."""
    if n_min < 1:
        raise DimensionError("n_min must be >= 1")
    if b.ndim != len(t):
        raise DimensionError("rhs order does not match coefficient count")
    for m, tm in enumerate(t):
        if tm.shape != (b.shape[m], b.shape[m]) or not is_upper_quasi_triangular(tm):
            raise DimensionError(f"coefficient {m} must be upper quasi-triangular")
    all_tri = all(np.all(np.tril(tm, -1) == 0) for tm in t)
    return _lap_rec(t, [(0, tm.shape[0]) for tm in t], np.asfortranarray(b, dtype=np.float64),
                    n_min, all_tri)


# ---- gsylv recursion (gsylv.hpp:62-159) -------------------------------------------------
def _gsylv_base(a, c, win, b, all_tri):
    """gsylv.hpp:70-94: kron(A_{d-1},...,A_1, C) window + I (x) A_0."""
    lo0, hi0 = win[0]
    op = c[lo0:hi0, lo0:hi0].copy()
    for m in range(1, len(win)):
        lo, hi = win[m]
        op = np.kron(a[m][lo:hi, lo:hi], op)
    n0 = hi0 - lo0
    a0 = a[0][lo0:hi0, lo0:hi0]
    for r in range(b.size // n0):
        op[r * n0:(r + 1) * n0, r * n0:(r + 1) * n0] += np.triu(a0, -1)
    vec = b.reshape(-1, order="F")
    sol = block_back_substitution(op, vec, None if all_tri else lower_block_partition(op))
    return sol.reshape(b.shape, order="F")


def _gs_rec(a, c, win, b, n_min, all_tri):
    """gsylv.hpp:96-128 with the two update cases."""
    mu, k = _pick_split(a, win, n_min)
    if mu < 0:
        return _gsylv_base(a, c, win, b, all_tri)
    lo, hi = win[mu]
    d = len(win)
    sl1 = [slice(None)] * d
    sl2 = [slice(None)] * d
    sl1[mu] = slice(0, k - lo)
    sl2[mu] = slice(k - lo, None)
    b1, b2 = b[tuple(sl1)].copy(), b[tuple(sl2)].copy()
    w2 = list(win)
    w2[mu] = (k, hi)
    x2 = _gs_rec(a, c, w2, b2, n_min, all_tri)
    wb = lambda m_, w: m_[w[0]:w[1], w[0]:w[1]]
    if mu == 0:  # gsylv.hpp:111-116
        b1 -= mode_multiply(x2, a[0][lo:k, k:hi], 0)
        t = mode_multiply(x2, c[lo:k, k:hi], 0)
        for m in range(1, d):
            t = mode_multiply(t, wb(a[m], win[m]), m)
        b1 -= t
    else:  # gsylv.hpp:117-123
        t = mode_multiply(x2, a[mu][lo:k, k:hi], mu)
        t = mode_multiply(t, wb(c, win[0]), 0)
        for m in range(1, d):
            if m != mu:
                t = mode_multiply(t, wb(a[m], win[m]), m)
        b1 -= t
    w1 = list(win)
    w1[mu] = (lo, k)
    x1 = _gs_rec(a, c, w1, b1, n_min, all_tri)
    return np.concatenate([x1, x2], axis=mu)


def gsylv_recursive(t: list, c: np.ndarray, b: np.ndarray, n_min: int) -> np.ndarray:
    """gsylv.hpp:149-159 (require_reduced_gsylv :130-141)."""
    if len(t) < 2:
        raise DimensionError("need at least two modes")
    if np.any(np.tril(c, -1) != 0):
        raise DimensionError("C must be upper triangular")
    for m, tm in enumerate(t):
        if tm.shape != (b.shape[m], b.shape[m]) or not is_upper_quasi_triangular(tm):
            raise DimensionError(f"coefficient {m} must be upper quasi-triangular")
    all_tri = all(np.all(np.tril(tm, -1) == 0) for tm in t)
    return _gs_rec(t, c, [(0, tm.shape[0]) for tm in t], np.asfortranarray(b, dtype=np.float64),
                   n_min, all_tri)


# ---- pipelines (laplace.hpp:248-302, gsylv.hpp:236-302), real arithmetic --------------------
def schur(a):
    """kernels.hpp:78-93 (dgees): A = U T U^T, T real quasi-triangular."""
    import scipy.linalg as sl
    t, u = sl.schur(np.asarray(a, dtype=np.float64), output="real")
    return u, t


def qz(a, c):
    """kernels.hpp:113-133 (dgges): A = Q S Z^T, C = Q T Z^T."""
    import scipy.linalg as sl
    s, t, q, z = sl.qz(np.asarray(a, dtype=np.float64), np.asarray(c, dtype=np.float64),
                       output="real")
    return q, z, s, t


def solve_laplace(coeffs, rhs, n_min=3):
    """laplace.hpp:248-302 with Strategy::recursion_only + real arithmetic."""
    f = [schur(a) for a in coeffs]
    bt = rhs
    for m, (u, _) in enumerate(f):
        bt = mode_multiply(bt, u.T, m)
    xt = laplace_recursive([t for _, t in f], bt, n_min)
    for m, (u, _) in enumerate(f):
        xt = mode_multiply(xt, u, m)
    return xt


def solve_gsylv(coeffs, c, rhs, n_min=3):
    """gsylv.hpp:236-302 with Strategy::recursion_only + real arithmetic."""
    q, z, s, tc = qz(coeffs[0], c)
    f = [schur(a) for a in coeffs[1:]]
    bt = mode_multiply(rhs, q.T, 0)
    for m, (u, _) in enumerate(f, start=1):
        bt = mode_multiply(bt, u.T, m)
    xt = gsylv_recursive([s] + [t for _, t in f], tc, bt, n_min)
    xt = mode_multiply(xt, z, 0)
    for m, (u, _) in enumerate(f, start=1):
        xt = mode_multiply(xt, u, m)
    return xt


# ---- dense oracle and residual (oracle.hpp:41-268) ----------------------------------------
def assemble_laplace(coeffs) -> np.ndarray:
    """oracle.hpp:41-74: sum_m I (x) ... A_m ... (x) I, A_0 on the fastest index."""
    dims = [a.shape[0] for a in coeffs]
    n = int(np.prod(dims))
    op = np.zeros((n, n))
    for m, a in enumerate(coeffs):
        left = int(np.prod(dims[:m]))
        right = int(np.prod(dims[m + 1:]))
        op += np.kron(np.eye(right), np.kron(a, np.eye(left)))
    return op


def assemble_gsylv(coeffs, c) -> np.ndarray:
    """oracle.hpp:78-129: I (x) ... (x) A_0 + A_{d-1} (x) ... (x) A_1 (x) C."""
    dims = [a.shape[0] for a in coeffs]
    n = int(np.prod(dims))
    k = c
    for a in coeffs[1:]:
        k = np.kron(a, k)
    return np.kron(np.eye(n // dims[0]), coeffs[0]) + k


def dense_solve_laplace(coeffs, rhs):
    return np.linalg.solve(assemble_laplace(coeffs), rhs.reshape(-1, order="F")).reshape(
        rhs.shape, order="F")


def dense_solve_gsylv(coeffs, c, rhs):
    return np.linalg.solve(assemble_gsylv(coeffs, c), rhs.reshape(-1, order="F")).reshape(
        rhs.shape, order="F")


def residual_laplace(coeffs, rhs, x) -> float:
    """oracle.hpp:233-247."""
    r = rhs.copy()
    scale = 0.0
    for m, a in enumerate(coeffs):
        r = r - mode_multiply(x, a, m)
        scale += np.linalg.norm(a)
    den = scale * np.linalg.norm(x) + np.linalg.norm(rhs)
    return float(np.linalg.norm(r) / den) if den else 0.0


def residual_gsylv(coeffs, c, rhs, x) -> float:
    """oracle.hpp:249-268."""
    r = rhs - mode_multiply(x, coeffs[0], 0)
    t = mode_multiply(x, c, 0)
    prod = 1.0
    for m in range(1, len(coeffs)):
        t = mode_multiply(t, coeffs[m], m)
        prod *= np.linalg.norm(coeffs[m])
    r = r - t
    den = (np.linalg.norm(coeffs[0]) + np.linalg.norm(c) * prod) * np.linalg.norm(x) + np.linalg.norm(rhs)
    return float(np.linalg.norm(r) / den) if den else 0.0


def min_kron_sum(eigs: list):
    """solvability.hpp:31-57: smallest |sum| over all tuples, first minimum in
    odometer order (mode 0 fastest); returns (min_abs, witness)."""
    grids = np.meshgrid(*[np.asarray(e) for e in eigs], indexing="ij")
    s = sum(grids)
    flat = np.abs(s).reshape(-1, order="F")
    i = int(np.argmin(flat))  # argmin returns the first occurrence
    idx = np.unravel_index(i, s.shape, order="F")
    return float(flat[i]), [int(v) for v in idx]


def quasi_tri_eigenvalues(t) -> list:
    """kernels.hpp:309-330."""
    n = t.shape[0]
    out, j = [], 0
    while j < n:
        if j + 1 < n and t[j + 1, j] != 0:
            tr = complex(t[j, j] + t[j + 1, j + 1]) / 2
            det = complex(t[j, j] * t[j + 1, j + 1] - t[j, j + 1] * t[j + 1, j])
            disc = np.sqrt(tr * tr - det)
            out += [tr + disc, tr - disc]
            j += 2
        else:
            out.append(complex(t[j, j]))
            j += 1
    return out
