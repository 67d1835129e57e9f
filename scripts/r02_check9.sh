#!/bin/bash
OUT=${OUT:-gpurun_out/r02_c9}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_momentum.py -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
B="--steps 30 --warmup 5 --no-variants --no-e2e --no-cpu-baseline"
for T in 8 16 32; do
  timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T $B > $OUT/mom_bf16_tau$T.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_commit_momentum -s 3 -c 1 \
   -o $OUT/ncu_mom_bf16_tau32 -f python bench.py --dtype bf16 --gamma 0.9 --tau 32 --steps 2 --warmup 3 --no-variants --no-e2e --no-cpu-baseline > $OUT/ncu_mom.log 2>&1
