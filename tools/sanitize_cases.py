"""Small solves through every kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck; tools/sanitize.sh).  Each case checks the
device residual so a sanitizer-perturbed schedule that gives a wrong answer
also fails.  Under the sanitizer the plans detect the serialising tool and
run the plain kernel order (plan.cpp `serialized`)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_09539_b200 as T  # noqa: E402

CFG = T.SolverConfig(strategy=T.Strategy.recursion_only, arithmetic=T.Arithmetic.real_quasitriangular)
CASES = [
    # (name, kind, dims, env)
    ("lap3 8^3 tiles (C1-type)", 1, (24, 20, 16), {"TSG_DECOUPLE": "0"}),
    ("lap16 TMA tiles (C2/C4-type)", 2, (36, 34, 33), {"TSG_LAP16": "1", "TSG_DECOUPLE": "0"}),
    ("lapd order 6 (C3-type)", 2, (5, 4, 4, 3, 3, 3), {"TSG_DECOUPLE": "0"}),
    ("decoupled fibre, register kernel", 2, (12, 10, 8), {}),
    ("decoupled fibre, DMMA-blocked kernel", 2, (16, 40, 33), {}),
    ("small-mode fused passes", 2, (24, 24, 16, 16), {}),
    ("gsylv gsyd (C5-type)", 5, (20, 4, 4, 4), {}),
]


def main() -> int:
    only = sys.argv[1:]
    bad = 0
    for name, kind, dims, env in CASES:
        if only and not any(o in name for o in only):
            continue
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            p = T.make_problem(kind, dims, seed=7)
            rep = T.solve_gsylv(p, CFG) if kind == 5 else T.solve_laplace(p, CFG)
            res = T.residual(p, rep.solution)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        ok = res < 1e-12
        bad += not ok
        print(f"{'ok ' if ok else 'BAD'} {name} {dims}: residual {res:.2e}", flush=True)
    # the transform GEMM alone (tsg_mode_multiply), odd shapes
    x = np.asfortranarray(np.random.default_rng(1).standard_normal((70, 33, 9)))
    a = np.asfortranarray(np.random.default_rng(2).standard_normal((40, 33)))
    y = T.mode_multiply(x, a, 1)
    want = np.einsum("ij,ajb->aib", a, x)
    e = float(np.abs(y - want).max())
    print(f"{'ok ' if e < 1e-12 else 'BAD'} mode_multiply (70,33,9) x_1 40x33: max err {e:.1e}", flush=True)
    bad += not e < 1e-12
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
