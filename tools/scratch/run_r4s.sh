#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
SETTINGS="RFR_T2FDYN=0 RFR_T2FDYN=1" tools/ab_env2.sh $TAG/c3
SETTINGS="RFR_T2FDYN=0 RFR_T2FDYN=1" BENCH_ARGS="--dense" tools/ab_env2.sh $TAG/dense
SETTINGS="RFR_T2FDYN=0 RFR_T2FDYN=1" BENCH_ARGS="--config c4" tools/ab_env2.sh $TAG/c4
SETTINGS="RFR_T2FDYN=0 RFR_T2FDYN=1" BENCH_ARGS="--step heatmap" tools/ab_env2.sh $TAG/heatmap
SETTINGS="RFR_T2FDYN=0 RFR_T2FDYN=1" BENCH_ARGS="--emulate-world 8 --emulate-rank 0" tools/ab_env2.sh $TAG/emu8
SETTINGS="RFR_T2FDYN=0 RFR_T2FDYN=1" BENCH_ARGS="--config c4 --emulate-world 8 --emulate-rank 0" tools/ab_env2.sh $TAG/c4emu8
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
