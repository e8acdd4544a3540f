#!/bin/bash
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02c}; cfg=${2:-C2}; k=${3:-fibre_wide}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
  -o $o/${t}_${k}_${cfg} -f python tools/perf_probe.py $cfg --reps 2 > $o/${t}_ncu_${k}_${cfg}.log 2>&1
echo done
