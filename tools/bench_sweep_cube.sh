# Interleaved bench sweep over the trailing-cube size / grid (development).
# usage (under gpurun): [CFG=C2] [STEPS=40] bash tools/bench_sweep_cube.sh "0 16" "6 16" ...
export PYTHONPATH=.
cfg=${CFG:-C2}
for r in 1 2; do
  for cg in "$@"; do
    read -r cube grid <<< "$cg"
    v=$(TSG_CUBE=$cube TSG_CUBE_GRID=$grid python bench.py --config $cfg --steps ${STEPS:-40} --no-cpu-baseline 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.4f %.4f %.4g' % (d['frac_fp64_peak_alg'], d['ms_per_step'], d['e2e']['value']))")
    echo "== r$r $cfg CUBE=$cube GRID=$grid $v"
  done
done
