#!/bin/bash
# each case in its own process (CUDA errors are sticky)
export PYTHONPATH=.
for dbg in ${DBGS:-0}; do
for dims in ${DIMSL:-"64,64,64"}; do
  r=$(TSG_LAP16=1 TSG_DBG=$dbg timeout 60 python - <<PY 2>&1 | tail -1
import numpy as np, paper_1905_09539_b200 as T
dims=($dims)
p=T.make_problem(2, dims, seed=1)
f=[T.schur(a) for a in p.coeffs]
from paper_1905_09539_b200.plan import Context, Plan
ctx=Context(0); pl=Plan(ctx,0,[x[1] for x in f],[x[0] for x in f])
x=np.zeros_like(p.rhs); rep=pl.execute_host(np.asfortranarray(p.rhs), x)
print("tiles", pl.info()["n_tiles"], "solve %.3f ms"%rep.t_solve_ms, "res %.2e"%T.residual(p, x))
PY
)
  echo "dbg=$dbg $dims: $r"
done; done
