#!/bin/bash
# run perf_probe against an alternative build of the library (experiments)
for f in "$@"; do
  cp paper_1905_09539_b200/libtsylv_gpu.so /tmp/lib_orig.so
  cp tools/alt/$f paper_1905_09539_b200/libtsylv_gpu.so
  echo "== $f"; PYTHONPATH=. TSG_VERBOSE=1 python tools/perf_probe.py C2 C4 --reps 2 2>&1 | grep -E "solve|grid" | sed -e "s/fwd.*solve/solve/" -e "s/back.*//" | sort -u
  cp /tmp/lib_orig.so paper_1905_09539_b200/libtsylv_gpu.so
done
