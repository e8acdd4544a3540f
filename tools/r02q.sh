export PYTHONPATH=.
t=$1; so=$2; cfgs=$3; pc=${4:-$3}
bash tools/r02_iter.sh $t "$cfgs"
cp tools/alt/$so paper_1905_09539_b200/libtsylv_gpu.so
TSG_PROF=1 timeout 300 python tools/perf_probe.py $pc --reps 2 > gpurun_out/${t}_prof.txt 2>&1
