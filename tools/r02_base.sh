#!/bin/bash
# Round-2 baseline GPU call: per-config timings, full GPU suite, bench + reference arm.
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $o/${t}_smi.txt
lscpu > $o/${t}_lscpu.txt
timeout 600 python tools/perf_probe.py C1 C2 C3 C4 C5 --reps 5 --check > $o/${t}_probe.txt 2>&1
TSG_DECOUPLE=0 timeout 600 python tools/perf_probe.py C2 C3 C4 --reps 5 > $o/${t}_probe_nodec.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > $o/${t}_pytest.log 2>&1; echo "pytest rc=$?" >> $o/${t}_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $o/${t}_bench.json 2> $o/${t}_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $o/${t}_ref.json 2> $o/${t}_ref.err
echo done
