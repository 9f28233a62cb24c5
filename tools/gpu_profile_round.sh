#!/bin/bash
# Round-end evidence in ONE GPU call (each ncu pass only after its command ran clean without ncu):
#   launch list of the bench command, full-size DRAM traffic of the hot kernels, ncu --set full of
#   K2 and of the fused K3/K4 sweep (first 2048 antennas of c3).
# usage: tools/gpu_profile_round.sh <tag>
set -u
TAG=${1:-prof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
BENCH="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 $BENCH > $OUT/bench_plain.jsonl 2> $OUT/bench_plain.err; echo "rc=$?" >> $OUT/bench_plain.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  $BENCH > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?" >> $OUT/ncu_launches.log
FULL="python tools/profile_step.py --config c3 --steps 1"
timeout 600 $FULL > $OUT/full_plain.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"${TRAFFIC_RX:-k_trace_fwd|k_adjoint|k_blend}" --csv --log-file $OUT/traffic.csv $FULL > $OUT/ncu_traffic.log 2>&1
echo "traffic rc=$?" >> $OUT/ncu_traffic.log
CMD="python tools/profile_step.py --config c3 --steps 2 --ants 2048"
timeout 600 $CMD > $OUT/profile_plain.log 2>&1 || { echo "plain run failed" >> $OUT/profile_plain.log; exit 0; }
i=0
for e in ${NCU_KERNELS:-k_trace_fwd:0 k_adjoint_tc:1}; do
  rx=${e%%:*}; sk=${e##*:}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$rx" -s $sk -c 1 -o $OUT/prof$i $CMD > $OUT/ncu_full$i.log 2>&1
  echo "ncu $rx rc=$?" >> $OUT/ncu_full$i.log
  i=$((i+1))
done
# (compute-sanitizer is closed on this GPU pool: memory safety is covered by the parity tests'
#  NaN-filled outputs, the small ragged cases and the workspace-region test instead)
