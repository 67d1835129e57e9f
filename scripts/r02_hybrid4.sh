#!/bin/bash
# Mixed transport with the copy engines taking the larger share (MLF_STAGE_SKIP=k: all remote
# operands but every k-th staged), 2 GPUs, configs 3 and 5.
OUT=${OUT:-gpurun_out/r02_hybrid4}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
timeout 600 env MLF_STAGE_SKIP=3 MLF_STAGE_FIRST_DIRECT=1 python -m pytest tests/test_gpu_multirank.py -q -k "staged_every" > $OUT/pytest_skip3.log 2>&1; echo "rc=$?" >> $OUT/pytest_skip3.log
run() {
  local name=$1; shift
  timeout 600 env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
     --master-port $((29900 + RANDOM % 500)) bench.py --gpus $NG --steps 10 --warmup 3 --no-e2e --no-variants \
     --no-cpu-baseline $BARGS > $OUT/$name.log 2>&1; echo rc=$? >> $OUT/$name.log
}
BARGS="--config 3 --mode fold" run fold_c3 MLF_X=0
for SK in 3 4; do
  for CH in 3 4 6; do
    BARGS="--config 3 --mode staged" run skip${SK}_ch${CH}_c3 MLF_STAGE_SKIP=$SK MLF_STAGE_CHUNKS=$CH MLF_STAGE_FIRST_DIRECT=1
  done
done
BARGS="--config 3 --mode staged" run e2_ch3_c3 MLF_STAGE_EVERY=2 MLF_STAGE_CHUNKS=3 MLF_STAGE_FIRST_DIRECT=1
