#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 300 python bench.py > $OUT/bench_c3.jsonl 2> $OUT/bench_c3.err
tools/scratch/run_configs.sh $TAG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
