export PYTHONPATH=.
for f in 1 2 3; do echo "== f=$f"; TSG_DECOUPLE_F=$f TSG_VERBOSE=1 timeout 300 python tools/perf_probe.py C3 --reps 3 --check 2>&1 | grep -E "decoupled solve|fwd|resid"; done > gpurun_out/r02zi_f.txt
