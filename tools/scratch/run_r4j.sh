#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 300 $B > $OUT/bench_c3.jsonl 2> $OUT/bench_c3.err
timeout 300 $B --dense > $OUT/bench_c3_dense.jsonl 2> $OUT/bench_c3_dense.err
timeout 300 $B --config c4 > $OUT/bench_c4.jsonl 2> $OUT/bench_c4.err
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
