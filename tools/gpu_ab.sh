#!/bin/bash
# A/B GPU call: selected tests, then bench variants given as "tag:ENV=..:args" entries in $VARIANTS.
# usage: TESTS="tests/x.py" VARIANTS="fused: sep::--separate" tools/gpu_ab.sh <tag>
set -u
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -n "${TESTS:-}" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest $TESTS -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
for v in ${VARIANTS:-}; do
  name=${v%%:*}; rest=${v#*:}; envs=${rest%%:*}; args=${rest#*:}
  env $(echo $envs | tr ',' ' ') timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline $args > $OUT/bench_$name.jsonl 2> $OUT/bench_$name.err
  echo "rc=$?" >> $OUT/bench_$name.err
done
