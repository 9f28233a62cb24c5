#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench.jsonl 2> $OUT/bench.err
RFR_T2FV=m6 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_m6.jsonl 2> $OUT/bench_m6.err
