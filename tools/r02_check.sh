#!/bin/bash
# GPU check: full test suite, the bench (C4 headline) and the reference arm.
export PYTHONPATH=.
o=gpurun_out; t=${1:-r02b}
python -m pytest tests -m gpu -x -q -s > $o/${t}_pytest.log 2>&1; echo "pytest rc=$?" >> $o/${t}_pytest.log
python bench.py --steps 20 --warmup 5 > $o/${t}_bench.json 2> $o/${t}_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $o/${t}_ref.json 2> $o/${t}_ref.err
echo done
