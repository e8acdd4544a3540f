export PYTHONPATH=.
for kb in 72 100 110; do echo "== smem $kb KB"; TSG_FIBRE_SMEM_KB=$kb TSG_VERBOSE=1 timeout 300 python tools/perf_probe.py C3 --reps 3 --check 2>&1 | grep -E "maxcol|fwd|resid"; done > gpurun_out/r02zo_sm.txt
