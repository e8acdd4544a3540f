#!/bin/bash
# One GPU call: bench line, ncu launch list of the same command, and
# ncu --set full captures of the solve and transform kernels (C2).
# usage (under gpurun): bash tools/profile_round.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
export PYTHONPATH=.
python bench.py --steps 40 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:solve_lap -s 2 -c 1 \
  -o gpurun_out/${tag}_solve_c2 -f python tools/perf_probe.py C2 --reps 4 > gpurun_out/${tag}_ncu_solve.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dgemm_nn -s 6 -c 1 \
  -o gpurun_out/${tag}_dgemm_c2 -f python tools/perf_probe.py C2 --reps 4 > gpurun_out/${tag}_ncu_dgemm.log 2>&1
echo done
