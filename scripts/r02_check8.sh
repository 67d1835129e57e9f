#!/bin/bash
OUT=${OUT:-gpurun_out/r02_c8}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_momentum.py tests/test_gpu_parity.py tests/test_sass_guard.py -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
B="--steps 20 --warmup 5 --no-variants --no-e2e --no-cpu-baseline"
for T in 4 8 16 32; do
  timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T $B > $OUT/mom_bf16_tau$T.log 2>&1
done
for SC in dynamic contig static; do
  for T in 4 32; do
    MLF_BULK_SCHED=$SC timeout 300 python bench.py --tau $T $B > $OUT/commit_f32_tau${T}_$SC.log 2>&1
  done
done
