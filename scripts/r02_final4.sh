#!/bin/bash
# Round-end 1-GPU check on the final build: the full GPU suite, smoke, the default bench line.
OUT=${OUT:-gpurun_out/r02_final10}
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.log 2>&1; echo "rc=$?" >> $OUT/bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_reference.log 2>&1; echo "rc=$?" >> $OUT/bench_reference.log
