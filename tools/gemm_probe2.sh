#!/bin/bash
for c in 1 6 7; do
  echo "cfg=$c"; TSG_GEMM_CFG=$c PYTHONPATH=. python tools/perf_probe.py C2 C4 C5 --reps 3 2>&1 | grep -E "fwd" | sed -e "s/solve.*back/back/" -e "s/total.*//"
done
cp paper_1905_09539_b200/libtsylv_gpu.so /tmp/orig.so; cp tools/alt/lib_st4.so paper_1905_09539_b200/libtsylv_gpu.so
for c in 1 6; do
  echo "4stage cfg=$c"; TSG_GEMM_CFG=$c PYTHONPATH=. python tools/perf_probe.py C2 C4 --reps 3 2>&1 | grep -E "fwd" | sed -e "s/solve.*back/back/" -e "s/total.*//"
done
cp /tmp/orig.so paper_1905_09539_b200/libtsylv_gpu.so
