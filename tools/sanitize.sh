#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over tools/sanitize_cases.py
# (one GPU; each tool bounded by its own timeout).  Output: gpurun_out/<tag>_sanitize_*.log
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02}
python tools/sanitize_cases.py > $o/${t}_sanitize_plain.log 2>&1; echo "rc=$?" >> $o/${t}_sanitize_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_cases.py > $o/${t}_sanitize_${tool}.log 2>&1
  echo "rc=$?" >> $o/${t}_sanitize_${tool}.log
done
echo done
