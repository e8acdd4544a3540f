#!/bin/bash
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02al}
timeout 600 python -m pytest tests/test_gpu_decoupled.py tests/test_gpu_repeat.py tests/test_gpu_dist_dec.py -x -q -p no:cacheprovider > $o/${t}_tests.log 2>&1; echo "rc=$?" >> $o/${t}_tests.log
timeout 300 python tools/perf_probe.py C1 C2 C3 C4 C5 --reps 5 --check > $o/${t}_probe.txt 2>&1
cp tools/alt/wprof.so paper_1905_09539_b200/libtsylv_gpu.so
TSG_PROF=1 timeout 300 python tools/perf_probe.py C3 --reps 2 > $o/${t}_prof.txt 2>&1
