#!/bin/bash
# Round-2 check 2: GPU test suite, momentum variants (wide vs 8-warp bf16 kernels, fp32).
OUT=${OUT:-gpurun_out/r02_c2}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
B="--steps 20 --warmup 5 --no-variants --no-e2e --no-cpu-baseline"
for T in 4 8 32; do
  timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T $B > $OUT/bench_bf16_mom_tau$T.log 2>&1
  MLF_MOM_WIDE=0 timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T $B > $OUT/bench_bf16_mom_tau${T}_8warp.log 2>&1
  timeout 300 python bench.py --dtype f32 --gamma 0.9 --tau $T $B > $OUT/bench_f32_mom_tau$T.log 2>&1
done
