#!/bin/bash
# Fused small-mode pass after the padded layout: tests, C3/C5 probe, ncu of the pass.
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02m}
mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_decoupled.py -m gpu -q -x -p no:cacheprovider -k "small or fuzz or decoupled" > $o/${t}_pytest.log 2>&1; echo "rc=$?" >> $o/${t}_pytest.log
timeout 600 python tools/perf_probe.py C3 C5 --reps 5 --check > $o/${t}_probe.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 1 -c 1 -o $o/${t}_pair_c3 -f python tools/perf_probe.py C3 --reps 2 > $o/${t}_ncu_pair_c3.log 2>&1
echo done
