#!/bin/bash
# Round-2 check 3: momentum A/B (one-member fast path on/off, 16- vs 8-warp bf16 kernel),
# planner latency on the box host, replica-trees tests, the bench line.
OUT=${OUT:-gpurun_out/r02_c3}
mkdir -p $OUT
B="--steps 20 --warmup 5 --no-variants --no-e2e --no-cpu-baseline"
for T in 4 8 16 32; do
  for SG in 1 0; do
    MLF_MOM_SINGLE=$SG timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T $B > $OUT/mom_bf16_tau${T}_single${SG}_wide.log 2>&1
    MLF_MOM_SINGLE=$SG MLF_MOM_WIDE=0 timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T $B > $OUT/mom_bf16_tau${T}_single${SG}_8warp.log 2>&1
    MLF_MOM_SINGLE=$SG timeout 300 python bench.py --dtype f32 --gamma 0.9 --tau $T $B > $OUT/mom_f32_tau${T}_single${SG}.log 2>&1
  done
done
for C in "4 8" "5 8" "3 8" "2 1"; do
  for T in 1 2 4 8; do
    MLF_PLAN_THREADS=$T timeout 300 python scripts/plan_time.py $C >> $OUT/plan_time.log 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_replica_trees.py tests/test_gpu_momentum.py tests/test_gpu_parity.py -q -x > $OUT/pytest_subset.log 2>&1; echo "rc=$?" >> $OUT/pytest_subset.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_default.log 2>&1
