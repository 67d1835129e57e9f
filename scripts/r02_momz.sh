#!/bin/bash
# bf16 momentum with exact packed products (FFMA2 with a -0 addend) + packed adds: bitwise and
# plain-definition tests, bench at tau 8/16/32 (MLF_MOM_WIDE=6 default), ncu of tau 32.
OUT=${OUT:-gpurun_out/r02_momz}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_momentum.py tests/test_sass_guard.py -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "momentum or bf16" > $OUT/pytest_parity.log 2>&1; echo "rc=$?" >> $OUT/pytest_parity.log
B="--steps 30 --warmup 5 --no-variants --no-e2e --no-cpu-baseline"
for r in 1 2; do
for T in 4 8 16 32; do
  timeout 300 python bench.py --dtype bf16 --gamma 0.9 --tau $T $B > $OUT/mom_bf16_tau${T}_r$r.log 2>&1
done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_commit_momentum -s 3 -c 1 \
   -o $OUT/ncu_mom_bf16_tau32 -f python bench.py --dtype bf16 --gamma 0.9 --tau 32 --steps 2 --warmup 3 --no-variants --no-e2e --no-cpu-baseline > $OUT/ncu_mom.log 2>&1
