#!/bin/bash
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02c}
timeout 900 python -m pytest tests/test_gpu_decoupled.py -x -q -s > $o/${t}_dec.log 2>&1; echo "rc=$?" >> $o/${t}_dec.log
TSG_VERBOSE=1 python tools/perf_probe.py C1 C2 C3 C4 --reps 5 --check > $o/${t}_probe.txt 2>&1
TSG_DECOUPLE=0 python tools/perf_probe.py C2 C4 --reps 3 > $o/${t}_probe_tile.txt 2>&1
timeout 600 ncu --set full --metrics smsp__pipe_tensor_subpipe_dmma_cycles_active,sm__inst_executed_pipe_tensor_subpipe_dmma --clock-control none --import-source on -k regex:fibre -s 1 -c 1 \
  -o $o/${t}_fibre_c3 -f python tools/perf_probe.py C3 --reps 2 > $o/${t}_ncu_fibre.log 2>&1
timeout 600 ncu --set full --metrics smsp__pipe_tensor_subpipe_dmma_cycles_active,sm__inst_executed_pipe_tensor_subpipe_dmma --clock-control none --import-source on -k regex:fibre -s 1 -c 1 \
  -o $o/${t}_fibre_c2 -f python tools/perf_probe.py C2 --reps 2 > $o/${t}_ncu_fibre2.log 2>&1
echo done
