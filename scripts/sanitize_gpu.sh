#!/bin/bash
# One compute-sanitizer tool per call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck
TOOL=${TOOL:-memcheck}
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
python -m pytest tests/test_gpu_parity.py -q -x -k "degenerate or longer or (random_plans and 0-bulk)" > $OUT/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --error-exitcode 99 --print-limit 20 \
   python -m pytest tests/test_gpu_parity.py -q -x -k "degenerate or longer or (random_plans and 0-bulk)" > $OUT/san_$TOOL.log 2>&1
echo "rc=$?" >> $OUT/san_$TOOL.log
