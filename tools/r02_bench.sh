#!/bin/bash
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02w}
timeout 900 python bench.py --steps 20 --warmup 5 > $o/${t}_bench.json 2> $o/${t}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${t}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-all-configs > $o/${t}_ncu_launch.log 2>&1
echo done
