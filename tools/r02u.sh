#!/bin/bash
# chunked sharded pipeline: dist tests, N=1 sharded bench with 1 and 4 chunks
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02u}
timeout 900 python -m pytest tests/test_gpu_dist_dec.py -x -q -p no:cacheprovider > $o/${t}_dist.log 2>&1; echo "rc=$?" >> $o/${t}_dist.log
for k in 1 4; do
  timeout 600 python bench.py --sharded --chunks $k --config C4 --steps 10 --warmup 3 --no-cpu-baseline > $o/${t}_shard_C4_k$k.json 2> $o/${t}_shard_C4_k$k.err
  echo "k=$k rc=$?" >> $o/${t}_shard_rc.txt
done
echo done
