#!/bin/bash
# One GPU call: parity tests, bench, ncu launch list, ncu --set full of the top kernels.
# usage: tools/gpu_round.sh <tag> [pytest-args]
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 python tools/profile_step.py --config c3 --steps 2 > $OUT/profile_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file $OUT/launches.csv python tools/profile_step.py --config c3 --steps 2 > $OUT/ncu_launches.log 2>&1
  echo "launches rc=$?" >> $OUT/ncu_launches.log
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_adjoint|k_trace_fwd|k_blend' \
     -s 5 -c 5 -o $OUT/prof python tools/profile_step.py --config c3 --steps 2 > $OUT/ncu_full.log 2>&1
  echo "full rc=$?" >> $OUT/ncu_full.log
fi
