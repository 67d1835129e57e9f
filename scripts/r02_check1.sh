#!/bin/bash
# Round-2 check: full GPU test suite, planner latency on the box host, bench (default + bf16
# momentum variants), ncu of the new bf16 momentum kernel.
OUT=${OUT:-gpurun_out/r02_c1}
mkdir -p $OUT
nproc > $OUT/host.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for C in "4 8" "5 8" "3 8" "2 1"; do
  for T in 1 4 8 16; do
    MLF_PLAN_THREADS=$T timeout 300 python scripts/plan_time.py $C >> $OUT/plan_time.log 2>&1
  done
done
for T in 4 8 32; do
  timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T --steps 20 --warmup 5 --no-variants --no-e2e --no-cpu-baseline > $OUT/bench_bf16_mom_tau$T.log 2>&1
done
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_default.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_commit_momentum -s 3 -c 1 \
   -o $OUT/ncu_mom_bf16_tau32_wide -f python bench.py --dtype bf16 --gamma 0.9 --tau 32 --steps 2 --warmup 3 --no-variants --no-e2e --no-cpu-baseline > $OUT/ncu_mom.log 2>&1
