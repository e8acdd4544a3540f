#!/bin/bash
# Round-2 first GPU call: per-config timings, ncu metric names for the
# FP64 tensor (DMMA) pipe, ncu --set full of the C3 / C5 solve kernels.
export PYTHONPATH=.
o=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $o/r02a_smi.txt
lscpu > $o/r02a_lscpu.txt
python tools/perf_probe.py C1 C2 C3 C4 C5 --reps 5 --check > $o/r02a_all.txt 2>&1
ncu --query-metrics --chip gb100 > $o/r02a_metrics_all.txt 2>&1
ncu --query-metrics-mode suffix --metrics sm__inst_executed_pipe_fp64,sm__pipe_fp64_cycles_active --chip gb100 > $o/r02a_metrics_fp64.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:solve_lapd -s 1 -c 1 \
  -o $o/r02a_lapd_c3 -f python tools/perf_probe.py C3 --reps 2 > $o/r02a_ncu_lapd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:solve_gsyd -s 1 -c 1 \
  -o $o/r02a_gsyd_c5 -f python tools/perf_probe.py C5 --reps 2 > $o/r02a_ncu_gsyd.log 2>&1
echo done
