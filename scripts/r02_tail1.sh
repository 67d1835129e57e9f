#!/bin/bash
# Bulk commit with the last wave in quarter tiles (MLF_BULK_TAIL=1, default) vs whole tiles (0):
# the bulk GPU tests, then config 2 at tau 4 (no split: 80 KB tiles) and tau 32 (528 KB tiles).
OUT=${OUT:-gpurun_out/r02_tail1}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "tail or tiles or dynamic or config2 or concurrent or contiguous" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for rep in 1 2; do
  for TL in 0 1; do
    for T in 4 32; do
      echo "== tail $TL tau $T rep $rep" >> $OUT/bench.log
      MLF_BULK_TAIL=$TL timeout 300 python bench.py --tau $T --steps 30 --warmup 5 --no-variants --no-e2e --no-cpu-baseline 2>&1 \
        | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $OUT/bench.log
    done
  done
done
