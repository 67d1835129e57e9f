#!/bin/bash
# Config 4 at N GPUs: the bulk commit's tile size (MLF_BULK_TILE) under NVLink-bound fold.
OUT=${OUT:-gpurun_out/r02_tile4}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
run() {
  local name=$1; shift
  timeout 600 env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
     --master-port $((29900 + RANDOM % 500)) bench.py --gpus $NG --steps 10 --warmup 3 --no-e2e --no-variants \
     --no-cpu-baseline $BARGS > $OUT/$name.log 2>&1; echo rc=$? >> $OUT/$name.log
}
for rep in 1 2; do
  for T in 0 1024 2048 4096; do
    BARGS="--config 4 --mode fold" run c4_tile${T}_r$rep MLF_BULK_TILE=$T
  done
done
