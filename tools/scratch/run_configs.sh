#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $B --dense > $OUT/bench_c3_dense.jsonl 2> $OUT/bench_c3_dense.err
for c in c1 c2 c4 c5; do timeout 900 $B --config $c > $OUT/bench_$c.jsonl 2> $OUT/bench_$c.err; done
for n in 2 4 8; do
  timeout 600 $B --emulate-world $n --emulate-rank 0 > $OUT/bench_emu_c3_N$n.jsonl 2> $OUT/bench_emu_c3_N$n.err
  timeout 900 $B --config c4 --emulate-world $n --emulate-rank 0 > $OUT/bench_emu_c4_N$n.jsonl 2> $OUT/bench_emu_c4_N$n.err
done
timeout 600 $B --step heatmap > $OUT/bench_c3_heatmap.jsonl 2> $OUT/bench_c3_heatmap.err
