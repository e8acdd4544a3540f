export PYTHONPATH=.
cp tools/alt/wprof.so paper_1905_09539_b200/libtsylv_gpu.so
TSG_PROF=1 timeout 300 python tools/perf_probe.py C2 --reps 2 > gpurun_out/${1}_prof.txt 2>&1
