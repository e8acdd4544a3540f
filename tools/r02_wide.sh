#!/bin/bash
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02b}
timeout 900 python -m pytest tests/test_gpu_decoupled.py -x -q -s -p no:cacheprovider > $o/${t}_dec.log 2>&1; echo "rc=$?" >> $o/${t}_dec.log
timeout 600 python tools/perf_probe.py C1 C2 C3 C4 --reps 5 --check > $o/${t}_probe.txt 2>&1
TSG_FIBRE_WIDE=0 timeout 300 python tools/perf_probe.py C1 C2 --reps 3 > $o/${t}_probe_big.txt 2>&1
bash tools/sanitize.sh $t
echo done
