#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc_gemm.py -m gpu -q > $OUT/pytest_tc.log 2>&1; echo "rc=$?" >> $OUT/pytest_tc.log
NCU_KERNELS="k2_filter k2_bwd k2_fwd k2_fout k2_cprep k2_gexp_tc k2_bins_tc" bash tools/gpu_profile_r2.sh $TAG
