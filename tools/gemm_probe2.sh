#!/bin/bash
# transform GEMM tile configurations (TSG_GEMM_CFG, gemm.cu dgemm_nn)
for c in ${CFGS_G:-1 2 3 4 6 7}; do
  echo "cfg=$c $(TSG_GEMM_CFG=$c PYTHONPATH=. python tools/perf_probe.py C2 C4 --reps 3 2>&1 | grep -E "fwd" | sed -e "s/solve.*back/back/" -e "s/total.*//" | tr -s ' ' | tr '\n' '|')"
done
