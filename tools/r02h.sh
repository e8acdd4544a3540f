export PYTHONPATH=.
t=${1:-r02h}
bash tools/r02_iter.sh $t "C1 C2 C4"
cp tools/alt/wprof.so paper_1905_09539_b200/libtsylv_gpu.so
TSG_PROF=1 timeout 300 python tools/perf_probe.py C2 C4 --reps 2 > gpurun_out/${t}_prof.txt 2>&1
