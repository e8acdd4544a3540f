#!/bin/bash
# Round-2 re-entry check at HEAD: smoke, full GPU suite, all-config probe,
# bench (C4 headline), reference arm, launch list.
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02h}
mkdir -p $o
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${t}_smoke.log 2>&1; echo "smoke rc=$?" >> $o/${t}_smoke.log
timeout 600 python tools/perf_probe.py C1 C2 C3 C4 C5 --reps 5 --check > $o/${t}_probe.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $o/${t}_pytest.log 2>&1; echo "pytest rc=$?" >> $o/${t}_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $o/${t}_bench.json 2> $o/${t}_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $o/${t}_ref.json 2> $o/${t}_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${t}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-all-configs > $o/${t}_ncu_launch.log 2>&1
echo done
