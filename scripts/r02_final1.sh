#!/bin/bash
# Round-2 final evidence on one GPU: planner timings, GPU tests + smoke, bench line, and the
# ncu launch list + one --set full capture of the headline kernel (after the plain run exits 0).
OUT=${OUT:-gpurun_out/r02_final}
mkdir -p $OUT
OUT=$OUT/planbox bash scripts/r02_planbox.sh
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_default.log 2>&1; echo "rc=$?" >> $OUT/bench_default.log
OUT=$OUT bash scripts/profile_1gpu.sh
