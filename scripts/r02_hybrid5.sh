#!/bin/bash
# Mixed transport, copy engines taking 3/4 .. 7/8 of the remote operands (MLF_STAGE_SKIP=k), 2 or 3
# chunks, configs 3 and 5 at 2 GPUs; config 4 fold (rank-0 planning time with the round-end planner).
OUT=${OUT:-gpurun_out/r02_hybrid5}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
run() {
  local name=$1; shift
  timeout 600 env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
     --master-port $((29900 + RANDOM % 500)) bench.py --gpus $NG --steps 10 --warmup 3 --no-e2e --no-variants \
     --no-cpu-baseline $BARGS > $OUT/$name.log 2>&1; echo rc=$? >> $OUT/$name.log
}
BARGS="--config 4 --mode fold" run fold_c4 MLF_X=0
for rep in 1 2; do
  for SK in 4 6 8; do
    for CH in 2 3; do
      BARGS="--config 3 --mode staged" run skip${SK}_ch${CH}_c3_r$rep MLF_STAGE_SKIP=$SK MLF_STAGE_CHUNKS=$CH MLF_STAGE_FIRST_DIRECT=1
    done
  done
done
BARGS="--config 5 --mode staged" run skip4_ch3_c5 MLF_STAGE_SKIP=4 MLF_STAGE_CHUNKS=3 MLF_STAGE_FIRST_DIRECT=1
BARGS="--config 5 --mode fold" run fold_c5 MLF_X=0
