#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in "X=0" "RFR_T2FV=m4" "RFR_T2FV=u2" "RFR_T2FV=m4u2" "RFR_T2SPT=6" "RFR_T2SPT=8"; do
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $OUT/b_$v.jsonl 2> $OUT/b_$v.err
  python -c "
import json;d=json.loads(open('$OUT/b_$v.jsonl').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],3), round(d['sweeps_ms_per_step']['filter'],3))" >> $OUT/summary.txt 2>&1
done
