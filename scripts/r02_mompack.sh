#!/bin/bash
# bf16 momentum (gamma 0.9): the packed-sum fold (exact FFMA2 products + FADD2) for short operand
# lists vs the scalar-add fold; GPU momentum tests first (bitwise + plain definition).
OUT=${OUT:-gpurun_out/r02_mompack}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_momentum.py tests/test_sass_guard.py -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for rep in 1 2; do
for PM in 0 12 40; do
  for T in 8 16 32; do
    echo "== pack_max $PM tau $T rep $rep" >> $OUT/bench.log
    MLF_MOM_PACK_MAX=$PM timeout 300 python bench.py --gamma 0.9 --dtype bf16 --tau $T --steps 20 --warmup 5 \
      --no-variants --no-e2e --no-cpu-baseline 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $OUT/bench.log
  done
done
done
