#!/bin/bash
# transform-GEMM tile configurations on C2/C4 (forward + back transform times)
for c in 0 1 2 3 4 5; do
  echo "cfg=$c"; TSG_GEMM_CFG=$c PYTHONPATH=. python tools/perf_probe.py C2 C4 --reps 3 2>&1 | grep -E "fwd" | sed -e "s/solve.*back/back/" -e "s/total.*//"
done
