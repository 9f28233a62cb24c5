#!/bin/bash
# Round-2 evidence in one GPU call (each ncu pass only after its command ran clean without ncu):
#   1. launch list of the bench command (per-launch device times, serialised and cold-cache)
#   2. DRAM traffic of the r2 sweeps at full size (c3, all 16384 antennas)
#   3. ncu --set full of each r2 sweep on the first 4096 antennas of c3, with its SASS source page
# usage: tools/gpu_profile_r2.sh <tag>
set -u
TAG=${1:-r2prof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
BENCH="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 $BENCH > $OUT/bench_plain.jsonl 2> $OUT/bench_plain.err; echo "rc=$?" >> $OUT/bench_plain.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  $BENCH > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?" >> $OUT/ncu_launches.log
FULL="python tools/profile_step.py --config c3 --steps 1"
timeout 600 $FULL > $OUT/full_plain.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"k2_" --csv --log-file $OUT/traffic.csv $FULL > $OUT/ncu_traffic.log 2>&1
echo "traffic rc=$?" >> $OUT/ncu_traffic.log
CMD="python tools/profile_step.py --config c3 --steps 2 --ants 4096"
timeout 600 $CMD > $OUT/profile_plain.log 2>&1 || { echo "plain run failed" >> $OUT/profile_plain.log; exit 0; }
for k in ${NCU_KERNELS:-k2_filter k2_bwd k2_fwd k2_fout k2_cprep}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 0 -c 1 \
    -o $OUT/$k $CMD > $OUT/ncu_$k.log 2>&1
  echo "ncu $k rc=$?" >> $OUT/ncu_$k.log
  ncu -i $OUT/$k.ncu-rep --page source --csv --print-source sass > $OUT/${k}_source.csv 2>/dev/null
  # summaries written on the box; only the filter's report travels back (gpurun_out/ is capped at 64 MiB)
  (python tools/ncu_summary.py $OUT/$k.ncu-rep; python tools/sass_mix.py $OUT/${k}_source.csv) > $OUT/${k}_summary.txt 2>&1
  [ "$k" = "k2_filter" ] || rm -f $OUT/$k.ncu-rep
done
