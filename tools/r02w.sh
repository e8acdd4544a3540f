#!/bin/bash
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02w}
timeout 600 python -m pytest tests/test_gpu_decoupled.py tests/test_gpu_complex.py -x -q -p no:cacheprovider > $o/${t}_dec.log 2>&1; echo "rc=$?" >> $o/${t}_dec.log
timeout 600 python tools/perf_probe.py C1 C2 C4 C5 --reps 5 --check > $o/${t}_probe.txt 2>&1
timeout 600 python - > $o/${t}_zbench.txt 2>&1 <<'PY'
import json, bench
import paper_1905_09539_b200 as T
print(json.dumps(bench.complex_configs(T), indent=1))
PY
echo done
