#!/bin/bash
# final round-2 ncu --set full captures: register fibre kernel (C3) after the
# row-I/O change, the complex fibre and GEMM kernels (Z2)
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02ac}
timeout 300 python tools/perf_probe.py C3 --reps 3 --check > $o/${t}_probe.txt 2>&1 || exit 1
timeout 300 python tools/zprobe.py Z2 > $o/${t}_zprobe.txt 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fibre_small -s 1 -c 1 \
  -o $o/${t}_fibre_c3 -f python tools/perf_probe.py C3 --reps 2 > $o/${t}_ncu_fibre_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zfibre_kernel -s 9 -c 1 \
  -o $o/${t}_zfibre_z2 -f python tools/zprobe.py Z2 > $o/${t}_ncu_zfibre.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -s 4 -c 1 \
  -o $o/${t}_zgemm_z2 -f python tools/zprobe.py Z2 > $o/${t}_ncu_zgemm.log 2>&1
echo done
