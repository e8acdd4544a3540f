#!/bin/bash
# Tile-extent / solve-variant evidence: per variant, the
# solve kernel's time, DMMA-pipe utilisation, DRAM bytes; one ncu metric pass
# each (not --set full), plus CUDA-event timing without ncu.
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02ev}
M=gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
run() {  # name cfg env... (-- perf_probe args)
  local name=$1 cfg=$2; shift 2
  env "$@" timeout 300 python tools/perf_probe.py $cfg --reps 3 > $o/${t}_${name}_time.txt 2>&1
  env "$@" timeout 600 ncu --metrics $M --clock-control none -k regex:"solve|fibre|dgemm|pair" -c 40 --csv \
    --log-file $o/${t}_${name}_ncu.csv python tools/perf_probe.py $cfg --reps 1 > /dev/null 2>&1
}
run c2_decoupled C2 X=1
run c2_lap16 C2 TSG_DECOUPLE=0
run c2_lap3 C2 TSG_DECOUPLE=0 TSG_LAP16=0
run c3_decoupled C3 X=1
run c3_lapd C3 TSG_DECOUPLE=0
run c4_decoupled C4 X=1
run c4_lap16 C4 TSG_DECOUPLE=0
run c5_decoupled C5 X=1
run c5_gsyd C5 TSG_DECOUPLE=0
echo done
