#!/bin/bash
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02s}
for c in ${2:-C4 C1}; do
  timeout 600 python bench.py --sharded --config $c --steps 10 --warmup 3 --no-cpu-baseline > $o/${t}_shard_$c.json 2> $o/${t}_shard_$c.err
  echo "$c rc=$?" >> $o/${t}_shard_rc.txt
done
echo done
