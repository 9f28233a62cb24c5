#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
SETTINGS="RFR_T2FWM=4 RFR_T2FWM=5 RFR_T2FWM=6" tools/ab_env2.sh $TAG/c3
SETTINGS="RFR_T2FWM=4 RFR_T2FWM=5 RFR_T2FWM=6" BENCH_ARGS="--dense" tools/ab_env2.sh $TAG/dense
SETTINGS="RFR_T2FWM=4 RFR_T2FWM=5 RFR_T2FWM=6" BENCH_ARGS="--step heatmap" tools/ab_env2.sh $TAG/heatmap
SETTINGS="RFR_T2FWM=4 RFR_T2FWM=5 RFR_T2FWM=6" BENCH_ARGS="--config c4" tools/ab_env2.sh $TAG/c4
timeout 900 python -m pytest tests/test_gpu_mf_adjoint.py tests/test_gpu_training.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
