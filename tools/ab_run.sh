#!/bin/bash
# A/B timing of alternative library builds (tools/alt/*.so), interleaved,
# on the same box: perf_probe phase times per build.
cfgs=${CFGS:-C2}
cp paper_1905_09539_b200/libtsylv_gpu.so /tmp/lib_orig.so
for r in 1 2; do
  for f in "$@"; do
    cp tools/alt/$f paper_1905_09539_b200/libtsylv_gpu.so
    echo "== $f round $r: $(PYTHONPATH=. python tools/perf_probe.py $cfgs --reps 3 2>&1 | grep -E "solve" | sed -e "s/ (\([0-9.]*\) TF[a-z ]*)/(\1)/g" -e "s/total.*//" | tr -s ' ' | tr '\n' '|')"
  done
done
cp /tmp/lib_orig.so paper_1905_09539_b200/libtsylv_gpu.so
