#!/bin/bash
# Round-2 probe: bf16 momentum (gamma 0.9) bench lines at tau 4/8/32, ncu --set full of the
# tau-32 momentum commit, and the planner latency on the box's host.
OUT=${OUT:-gpurun_out/r02_mom}
mkdir -p $OUT
nproc > $OUT/host.txt; lscpu | grep "Model name" >> $OUT/host.txt
for T in 4 8 32; do
  timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T --steps 20 --warmup 5 --no-variants --no-e2e --no-cpu-baseline > $OUT/bench_bf16_mom_tau$T.log 2>&1
done
timeout 300 python bench.py --dtype f32 --gamma 0.9 --tau 32 --steps 20 --warmup 5 --no-variants --no-e2e --no-cpu-baseline > $OUT/bench_f32_mom_tau32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_commit_momentum -s 3 -c 1 \
   -o $OUT/ncu_mom_bf16_tau32 -f python bench.py --dtype bf16 --gamma 0.9 --tau 32 --steps 2 --warmup 3 --no-variants --no-e2e --no-cpu-baseline > $OUT/ncu_mom.log 2>&1
for C in "4 8" "5 8" "3 8" "2 1"; do
  MLF_PLAN_THREADS=$(nproc) timeout 300 python scripts/plan_time.py $C >> $OUT/plan_time.log 2>&1
  MLF_PLAN_THREADS=1 timeout 300 python scripts/plan_time.py $C >> $OUT/plan_time.log 2>&1
done
