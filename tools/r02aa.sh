#!/bin/bash
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02aa}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decoupled.py tests/test_gpu_fuzz.py tests/test_gpu_repeat.py -x -q -p no:cacheprovider > $o/${t}_tests.log 2>&1; echo "rc=$?" >> $o/${t}_tests.log
timeout 300 python tools/perf_probe.py C3 C5 --reps 5 --check > $o/${t}_probe.txt 2>&1
cp tools/alt/pprof.so paper_1905_09539_b200/libtsylv_gpu.so
TSG_PROF=1 timeout 300 python tools/perf_probe.py C3 C5 --reps 2 > $o/${t}_prof_bulk.txt 2>&1
TSG_PAIR_BULK=0 TSG_PROF=1 timeout 300 python tools/perf_probe.py C3 C5 --reps 2 > $o/${t}_prof_nobulk.txt 2>&1
echo done
