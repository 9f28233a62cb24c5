#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench1.jsonl 2> $OUT/bench1.err
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tools/scratch/run_configs.sh $TAG
