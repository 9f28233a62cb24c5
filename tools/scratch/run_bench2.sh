#!/bin/bash
set -u
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > $OUT/bench$i.jsonl 2> $OUT/bench$i.err; done
