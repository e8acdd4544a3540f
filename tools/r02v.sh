#!/bin/bash
# complex path: tests + the complex bench configs
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02v}
timeout 1200 python -m pytest tests/test_gpu_complex.py tests/test_gpu_cli.py tests/test_gpu_cpp_dropin.py -x -q -p no:cacheprovider > $o/${t}_z.log 2>&1; echo "rc=$?" >> $o/${t}_z.log
timeout 600 python - > $o/${t}_zbench.txt 2>&1 <<'PY'
import json, bench
import paper_1905_09539_b200 as T
print(json.dumps(bench.complex_configs(T), indent=1))
PY
echo done
