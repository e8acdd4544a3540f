#!/bin/bash
# Round-2 ncu --set full captures of the default-path kernels (one launch
# each, after the program ran clean without ncu): transform GEMM and team
# fibre kernel at C4, register fibre kernel and fused small-mode pass at C3,
# pencil team kernel at C5.
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02i}
mkdir -p $o
timeout 600 python tools/perf_probe.py C1 C2 C3 C4 C5 --reps 5 --check > $o/${t}_probe.txt 2>&1 || exit 1
cap() {  # tag config kernel-regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 \
    -o $o/${t}_$1 -f python tools/perf_probe.py $2 --reps 2 > $o/${t}_ncu_$1.log 2>&1
}
cap dgemm_c4 C4 dgemm_nn 1
cap fibre_c4 C4 fibre_wide 1
cap fibre_c3 C3 fibre_small 1
cap pair_c3 C3 pair_kernel 1
cap fibre_c5 C5 fibre_wide 1
cap dgemm_c2 C2 dgemm_nn 1
ls -la $o
echo done
