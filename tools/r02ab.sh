#!/bin/bash
# A/B of library variants (tools/alt/<name>.so): probe per variant
export PYTHONPATH=.
o=gpurun_out; t=$1; cfgs=$2; shift 2
timeout 300 python tools/perf_probe.py $cfgs --reps 5 --check > $o/${t}_base.txt 2>&1
for v in "$@"; do
  cp tools/alt/$v.so paper_1905_09539_b200/libtsylv_gpu.so
  timeout 300 python tools/perf_probe.py $cfgs --reps 5 --check > $o/${t}_$v.txt 2>&1
done
echo done
