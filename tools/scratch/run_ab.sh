#!/bin/bash
# usage: run_ab.sh <tag>
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_fullsize.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
RFR_T2GEO=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_geo0.jsonl 2> $OUT/bench_geo0.err
