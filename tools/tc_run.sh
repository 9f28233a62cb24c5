#!/bin/bash
OUT=gpurun_out/tc1; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "filter or backward or edge or comm or workspace or shard or reuse" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_tc.jsonl 2> $OUT/bench_tc.err
RFR_ADJOINT=simt timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_simt.jsonl 2> $OUT/bench_simt.err
