export PYTHONPATH=.
t=$1; so=${2:-wprof.so}; cfgs=${3:-C2}
cp tools/alt/$so paper_1905_09539_b200/libtsylv_gpu.so
TSG_PROF=1 timeout 300 python tools/perf_probe.py $cfgs --reps 2 > gpurun_out/${t}_prof.txt 2>&1
