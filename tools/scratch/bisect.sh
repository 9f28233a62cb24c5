#!/bin/bash
OUT=gpurun_out/bis; mkdir -p $OUT
T=tests/test_gpu_fullsize.py::test_r2_direct_node_evaluation_wide_global_spread
for v in "RFR_T2GEO=0" "RFR_T2TC=0" "RFR_T2GEO=2"; do
  env $v timeout 300 python -m pytest $T -q -x > $OUT/$v.log 2>&1; echo "$v rc=$?" >> $OUT/summary.txt
done
timeout 1500 python -m pytest tests -m gpu -q > $OUT/all.log 2>&1; echo "all rc=$?" >> $OUT/summary.txt
