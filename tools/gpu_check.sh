#!/bin/bash
# GPU call: selected pytest files, optional bench, and one ncu --set full capture per kernel listed
# (one kernel per ncu process: later kernels of a multi-kernel capture came back as nan).
# usage: TESTS="tests/x.py" BENCH=1 NCU_LIST="k_adjoint:1 k_trace_fwd:0" ANTS=2048 tools/gpu_check.sh <tag>
#   NCU_LIST entries are <regex>:<launch-skip among matching kernels>
set -u
TAG=${1:-chk}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -n "${TESTS:-}" ]; then
  timeout 1500 python -m pytest $TESTS -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
if [ "${BENCH:-0}" = "1" ]; then
  timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS:-} > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
fi
if [ -n "${NCU_LIST:-}" ]; then
  CMD="python tools/profile_step.py --config ${PCFG:-c3} --steps 2 --ants ${ANTS:-2048}"
  timeout 600 $CMD > $OUT/profile_plain.log 2>&1 || { echo "plain run failed" >> $OUT/profile_plain.log; exit 0; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
  i=0
  for e in $NCU_LIST; do
    rx=${e%%:*}; sk=${e##*:}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $sk -c 1 -o $OUT/prof$i $CMD > $OUT/ncu_full$i.log 2>&1
    echo "ncu $rx rc=$?" >> $OUT/ncu_full$i.log
    i=$((i+1))
  done
fi
