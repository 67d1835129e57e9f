#!/bin/bash
# Mixed transport at 4 GPUs with the copy engines taking a smaller share (MLF_STAGE_EVERY=k: every
# k-th remote operand staged), config 3; fold as the reference.
OUT=${OUT:-gpurun_out/r02_hybrid6}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
run() {
  local name=$1; shift
  timeout 600 env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
     --master-port $((29900 + RANDOM % 500)) bench.py --gpus $NG --steps 10 --warmup 3 --no-e2e --no-variants \
     --no-cpu-baseline $BARGS > $OUT/$name.log 2>&1; echo rc=$? >> $OUT/$name.log
}
BARGS="--config 3 --mode fold" run fold_c3 MLF_X=0
for EV in 3 4 6 8; do
  for CH in 3; do
    BARGS="--config 3 --mode staged" run every${EV}_ch${CH}_c3 MLF_STAGE_EVERY=$EV MLF_STAGE_CHUNKS=$CH MLF_STAGE_FIRST_DIRECT=1
  done
done
BARGS="--config 3 --mode staged" run every4_ch4_c3 MLF_STAGE_EVERY=4 MLF_STAGE_CHUNKS=4 MLF_STAGE_FIRST_DIRECT=1
BARGS="--config 3 --mode staged" run skip4_ch3_c3 MLF_STAGE_SKIP=4 MLF_STAGE_CHUNKS=3 MLF_STAGE_FIRST_DIRECT=1
