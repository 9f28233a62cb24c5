#!/bin/bash
# GPU call: selected pytest files + an ncu --set full capture of chosen kernels on a reduced config.
# usage: TESTS="tests/x.py" KREGEX='k_adjoint' ANTS=2048 tools/gpu_check.sh <tag>
set -u
TAG=${1:-chk}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -n "${TESTS:-}" ]; then
  timeout 1500 python -m pytest $TESTS -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
if [ "${BENCH:-0}" = "1" ]; then
  timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
fi
if [ -n "${KREGEX:-}" ]; then
  CMD="python tools/profile_step.py --config ${PCFG:-c3} --steps 2 --ants ${ANTS:-2048}"
  timeout 600 $CMD > $OUT/profile_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${SKIP:-0} -c ${COUNT:-4} -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
  echo "ncu rc=$?" >> $OUT/ncu_full.log
fi
