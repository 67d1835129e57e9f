#!/bin/bash
# bf16 momentum A/B: the 16-warp kernel (1 CTA/SM) vs two 8-warp CTAs per SM (MLF_MOM_BH2=1).
OUT=${OUT:-gpurun_out/r02_momb}
mkdir -p $OUT
MLF_MOM_BH2=1 timeout 900 python -m pytest tests/test_gpu_momentum.py -q > $OUT/pytest_bh2.log 2>&1; echo "rc=$?" >> $OUT/pytest_bh2.log
B="--steps 30 --warmup 5 --no-variants --no-e2e --no-cpu-baseline"
for r in 1 2; do
for T in 8 16 32; do
  timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T $B > $OUT/base_tau${T}_r$r.log 2>&1
  MLF_MOM_BH2=1 timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T $B > $OUT/bh2_tau${T}_r$r.log 2>&1
done
done
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_default.log 2>&1; echo "rc=$?" >> $OUT/bench_default.log
