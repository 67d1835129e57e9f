#!/bin/bash
OUT=${OUT:-gpurun_out/r02_c7}
mkdir -p $OUT
B="--steps 20 --warmup 5 --no-variants --no-e2e --no-cpu-baseline"
for T in 4 8 16 32; do
  timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T $B > $OUT/mom_bf16_tau$T.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_momentum.py tests/test_sass_guard.py -q > $OUT/pytest_momentum.log 2>&1; echo "rc=$?" >> $OUT/pytest_momentum.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_commit_momentum -s 3 -c 1 \
   -o $OUT/ncu_mom_bf16_tau32 -f python bench.py --dtype bf16 --gamma 0.9 --tau 32 --steps 2 --warmup 3 --no-variants --no-e2e --no-cpu-baseline > $OUT/ncu_mom.log 2>&1
