#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
for k in 5 10 20; do
  timeout 300 python bench.py --steps $k --warmup 3 --no-cpu-baseline > $OUT/bench_s$k.jsonl 2> $OUT/bench_s$k.err
done
timeout 300 python bench.py --steps 10 --warmup 3 > $OUT/bench_s10_cpu.jsonl 2> $OUT/bench_s10_cpu.err
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r4n/*.jsonl')):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d['steps'], round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['sweeps_ms_per_step'].items()})
PY
