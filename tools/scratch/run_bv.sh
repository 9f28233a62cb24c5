#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in "X=0" "RFR_T2BV=5" "RFR_T2BV=6" "RFR_T2FWM=4" "X=1"; do
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $OUT/b_$v.jsonl 2> $OUT/b_$v.err
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --dense > $OUT/d_$v.jsonl 2> $OUT/d_$v.err
  python -c "
import json
for f in ('b','d'):
  d=json.loads(open('$OUT/'+f+'_$v.jsonl').read().strip().splitlines()[-1]); s=d['sweeps_ms_per_step']
  print(f, '$v', round(d['ms_per_step'],3), 'bwd', round(s['backward'],3), 'fwd', round(s['forward'],3), 'flt', round(s['filter'],3))" >> $OUT/summary.txt 2>&1
done
