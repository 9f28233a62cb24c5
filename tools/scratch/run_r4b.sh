#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench$i.jsonl 2> $OUT/bench$i.err; done
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
