#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
SETTINGS="RFR_K1=thread RFR_K1=warp" tools/ab_env2.sh $TAG/c3
SETTINGS="RFR_K1=thread RFR_K1=warp" BENCH_ARGS="--emulate-world 8 --emulate-rank 0" tools/ab_env2.sh $TAG/emu8
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
