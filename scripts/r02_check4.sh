#!/bin/bash
# Round-2 check 4: fp32 momentum, this code vs the 27ddf8b build (scratch_old/), plus the read probe.
OUT=${OUT:-gpurun_out/r02_c4}
mkdir -p $OUT
B="--steps 20 --warmup 5 --no-variants --no-e2e --no-cpu-baseline"
for T in 4 32; do
  timeout 300 python bench.py --dtype f32 --gamma 0.9 --tau $T $B > $OUT/new_f32_tau$T.log 2>&1
  MLF_MOM_SINGLE=0 timeout 300 python bench.py --dtype f32 --gamma 0.9 --tau $T $B > $OUT/new_f32_tau${T}_single0.log 2>&1
  (cd scratch_old && timeout 300 python bench.py --dtype f32 --gamma 0.9 --tau $T $B > ../$OUT/old_f32_tau$T.log 2>&1)
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-variants --no-e2e --no-cpu-baseline > $OUT/new_default.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_commit_momentum -s 3 -c 1 \
   -o $OUT/ncu_f32_tau32_new -f python bench.py --dtype f32 --gamma 0.9 --tau 32 --steps 2 --warmup 3 --no-variants --no-e2e --no-cpu-baseline > $OUT/ncu_new.log 2>&1
(cd scratch_old && timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_commit_momentum -s 3 -c 1 \
   -o ../$OUT/ncu_f32_tau32_old -f python bench.py --dtype f32 --gamma 0.9 --tau 32 --steps 2 --warmup 3 --no-variants --no-e2e --no-cpu-baseline > ../$OUT/ncu_old.log 2>&1)
