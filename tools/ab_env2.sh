#!/bin/bash
# A/B of environment settings on the bench step; entries separated by spaces, variables of one
# entry by commas.  usage: SETTINGS="A=1,B=2 A=0" BENCH_ARGS="..." tools/ab_env2.sh <tag>
set -u
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for s in ${SETTINGS:-NONE=1}; do
  env ${s//,/ } timeout 300 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > $OUT/bench_$s.jsonl 2> $OUT/bench_$s.err
  python - "$s" "$OUT/bench_$s.jsonl" <<'PY' >> $OUT/summary.txt
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d["sweeps_ms_per_step"].items()})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
cat $OUT/summary.txt
