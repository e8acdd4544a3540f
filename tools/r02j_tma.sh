#!/bin/bash
# A/B of the TMA-staged transform GEMM (TSG_GEMM_TMA = 0 / 1 / 4) on one box.
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02j}
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_gemm_tma.py -m gpu -q -x -p no:cacheprovider > $o/${t}_pytest.log 2>&1; echo "rc=$?" >> $o/${t}_pytest.log
for r in 1 2; do
for v in 0 1 2 4; do
  echo "== TSG_GEMM_TMA=$v round $r" >> $o/${t}_probe.txt
  TSG_GEMM_TMA=$v timeout 600 python tools/perf_probe.py C1 C2 C4 C5 --reps 5 --check >> $o/${t}_probe.txt 2>&1
done
done
for v in 0 1; do
  TSG_GEMM_TMA=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dgemm --csv --log-file $o/${t}_launches_tma$v.csv python tools/perf_probe.py C2 C4 --reps 2 > $o/${t}_ncu_tma$v.log 2>&1
done
echo done
