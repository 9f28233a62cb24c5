#!/bin/bash
# quick TC-adjoint check: parity subset + A/B bench (tensor cores vs SIMT adjoint)
OUT=gpurun_out/${1:-tc}; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mf_adjoint.py -x -q -k "filter or backward or edge or comm or workspace or shard or reuse or adjoint" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_tc.jsonl 2> $OUT/bench_tc.err
if [ "${SIMT:-0}" = "1" ]; then RFR_ADJOINT=simt timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_simt.jsonl 2> $OUT/bench_simt.err; fi
if [ -n "${NCU_K:-}" ]; then
  CMD="python tools/profile_step.py --config c3 --steps 2 --ants 2048"
  timeout 300 $CMD > $OUT/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -s ${NCU_S:-1} -c 1 -o $OUT/prof $CMD > $OUT/ncu.log 2>&1
fi
