#!/bin/bash
# quick iteration: decoupled tests, probe, optional ncu of one kernel
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02x}; cfgs=${2:-"C1 C2 C3 C4"}; k=${3:-}; kc=${4:-C2}
timeout 300 python -m pytest tests/test_gpu_decoupled.py -x -q -s -p no:cacheprovider > $o/${t}_dec.log 2>&1; echo "rc=$?" >> $o/${t}_dec.log
timeout 300 python tools/perf_probe.py $cfgs --reps 5 --check > $o/${t}_probe.txt 2>&1
if [ -n "$k" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
  -o $o/${t}_${k}_${kc} -f python tools/perf_probe.py $kc --reps 2 > $o/${t}_ncu.log 2>&1
fi
echo done
