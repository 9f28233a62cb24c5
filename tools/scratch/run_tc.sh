#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python tools/scratch/tc_check.py > $OUT/tc_check.log 2>&1; echo "rc=$?" >> $OUT/tc_check.log
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
RFR_T2TC=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_simt.jsonl 2> $OUT/bench_simt.err
