#!/bin/bash
# Bulk commit last-wave quarter tiles (MLF_BULK_TAIL) at N GPUs: configs 3 and 4, fold.
OUT=${OUT:-gpurun_out/r02_tail4}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
run() {
  local name=$1; shift
  timeout 600 env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
     --master-port $((29900 + RANDOM % 500)) bench.py --gpus $NG --steps 10 --warmup 3 --no-e2e --no-variants \
     --no-cpu-baseline $BARGS > $OUT/$name.log 2>&1; echo rc=$? >> $OUT/$name.log
}
for rep in 1 2; do
  for TL in 0 1; do
    BARGS="--config 4 --mode fold" run c4_tail${TL}_r$rep MLF_BULK_TAIL=$TL
    BARGS="--config 3 --mode fold" run c3_tail${TL}_r$rep MLF_BULK_TAIL=$TL
  done
done
