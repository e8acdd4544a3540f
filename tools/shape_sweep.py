"""Default-path solves (no forcing) of a list of shapes through the public
API with the device residual, one process per shape under `timeout` by the
caller: a hang / correctness sweep of the kernel selection and the overlaps
(development).  usage: python tools/shape_sweep.py 208,200,256 [...]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_1905_09539_b200 as T  # noqa: E402

for arg in sys.argv[1:]:
    dims = tuple(int(v) for v in arg.split(","))
    p = T.make_problem(2, dims, seed=3)
    cfg = T.SolverConfig(strategy=T.Strategy.recursion_only, arithmetic=T.Arithmetic.real_quasitriangular)
    t = time.time()
    rep = T.solve_laplace(p, cfg)
    print(f"{dims} residual {rep.residual:.2e} {time.time() - t:.2f}s", flush=True)
    assert rep.residual < 1e-12
