"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref, the
unmodified tsylv headers built by oracle/Makefile).  Run here (where
/root/reference exists):  python tests/golden/make_golden.py
The .npz files are committed; nothing on the GPU box needs the reference."""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle.ref as R  # noqa: E402


def ref_baseline(kind, dims, seed):
    """BASELINE.json generators composed from the reference RandomStream
    (draw order: coefficients in mode order, then the rhs)."""
    rs = R.RandomStream(seed)
    if kind == 5:
        n0, nc = dims[0], dims[1]
        A = rs.randn(n0 * n0).reshape((n0, n0), order="F") / math.sqrt(n0) + 4 * np.eye(n0)
        B = rs.randn(n0 * n0).reshape((n0, n0), order="F") / math.sqrt(n0)
        C = rs.randn(nc * nc).reshape((nc, nc), order="F") / (2 * math.sqrt(nc))
        rhs = rs.randn(int(np.prod(dims))).reshape(dims, order="F")
        return [A] + [C.T.copy()] * (len(dims) - 1), B, rhs
    co = []
    for n in dims:
        if kind == 1:
            c = 0.5 + 1.5 * rs.uniform()
            h2, h1 = (n + 1) ** 2, c * (n + 1) / 2
            a = np.diag(np.full(n, 2.0 * h2)) + np.diag(np.full(n - 1, -h2 + h1), 1) + \
                np.diag(np.full(n - 1, -h2 - h1), -1)
            co.append(a)
        else:
            co.append(rs.randn(n * n).reshape((n, n), order="F") / math.sqrt(n) + 3 * np.eye(n))
    return co, None, rs.randn(int(np.prod(dims))).reshape(dims, order="F")


def pack(prefix, coeffs, out):
    for m, a in enumerate(coeffs):
        out[f"{prefix}_A{m}"] = a


def main():
    out = {}
    # RandomStream known answers (random.hpp:19-62)
    for seed in (1, 42, 987654321):
        rs = R.RandomStream(seed)
        out[f"rng{seed}_uniform"] = np.array([rs.uniform() for _ in range(16)])
        out[f"rng{seed}_normal"] = np.array([rs.normal() for _ in range(33)])
    # BASELINE-shaped instances, small: inputs + reference solutions
    cases = [("c1", 1, (12, 10, 8)), ("c2", 2, (12, 10, 8)), ("c3", 2, (4, 3, 3, 2, 3, 2)),
             ("c4", 2, (16, 8, 4)), ("c5", 5, (20, 4, 4, 4))]
    for name, kind, dims in cases:
        co, c, rhs = ref_baseline(kind, dims, 1)
        pack(name, co, out)
        out[f"{name}_rhs"] = rhs
        out[f"{name}_dims"] = np.array(dims)
        if kind == 5:
            out[f"{name}_C"] = c
            x, info = R.solve_gsylv(co, c, rhs)                      # default: merge+complex
            xr, infor = R.solve_gsylv(co, c, rhs, strategy=0, arithmetic=1, n_min=3)
        else:
            x, info = R.solve_laplace(co, rhs)
            xr, infor = R.solve_laplace(co, rhs, strategy=0, arithmetic=1, n_min=3)
        out[f"{name}_X_default"] = x
        out[f"{name}_X_real"] = xr
        out[f"{name}_residual"] = np.array([info[0], infor[0]])
    # reduced-form known answers (laplace_recursive / gsylv_recursive)
    rs = R.RandomStream(1001)
    for i, dims in enumerate([(4, 5), (3, 4, 5), (6, 3, 4, 2), (2, 3, 2, 2, 3)]):
        t, b = rs.reduced_laplace(list(dims))
        pack(f"lr{i}", t, out)
        out[f"lr{i}_B"] = b
        out[f"lr{i}_X"] = R.laplace_recursive(t, b, 2)
    rs = R.RandomStream(1002)
    t = [rs.quasi_triangular(n, 1.0, 0.6) for n in (7, 5, 6)]
    b = rs.randn(7 * 5 * 6).reshape((7, 5, 6), order="F")
    pack("lq", t, out)
    out["lq_B"] = b
    out["lq_X"] = R.laplace_recursive(t, b, 3)
    rs = R.RandomStream(2001)
    for i, dims in enumerate([(4, 5), (3, 4, 5), (5, 3, 4, 2)]):
        t, c, b = rs.reduced_gsylv(list(dims))
        pack(f"gr{i}", t, out)
        out[f"gr{i}_C"] = c
        out[f"gr{i}_B"] = b
        out[f"gr{i}_X"] = R.gsylv_recursive(t, c, b, 2)
    # mode products (tensor.hpp:187-231)
    rs = R.RandomStream(11)
    x = rs.randn(5 * 4 * 3).reshape((5, 4, 3), order="F")
    out["mm_X"] = x
    for m in range(3):
        a = rs.randn(6 * x.shape[m]).reshape((6, x.shape[m]), order="F")
        out[f"mm_A{m}"] = a
        out[f"mm_Y{m}"] = R.mode_multiply(x, a, m)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
