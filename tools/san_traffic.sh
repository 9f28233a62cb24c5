#!/bin/bash
# (1) compute-sanitizer memcheck on a small parity subset (one tool per call, per the profiling guide)
# (2) full-size c3 ncu --set full of K2 for the bench's roofline traffic (dram bytes per launch)
OUT=gpurun_out/${1:-san}; mkdir -p $OUT
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "c0a or c0b or edge_empty or edge_one or domain or workspace or comm" > $OUT/memcheck.log 2>&1; echo "memcheck rc=$?" >> $OUT/memcheck.log
CMD="python tools/profile_step.py --config c3 --steps 1"
timeout 600 $CMD > $OUT/plain.log 2>&1 && \
timeout 1200 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:"k_trace_fwd|k_adjoint" -c 3 -o $OUT/traffic $CMD > $OUT/ncu.log 2>&1
echo "ncu rc=$?" >> $OUT/ncu.log
