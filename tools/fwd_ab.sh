#!/bin/bash
OUT=gpurun_out/${1:-fwdab}; mkdir -p $OUT
RFR_FWD_B=16 timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mf_adjoint.py -x -q -k "forward or edge or adjoint or determinism" > $OUT/pytest16.log 2>&1; echo "rc=$?" >> $OUT/pytest16.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench32.jsonl 2> $OUT/bench32.err
RFR_FWD_B=16 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench16.jsonl 2> $OUT/bench16.err
