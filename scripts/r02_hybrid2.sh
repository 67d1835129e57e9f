#!/bin/bash
# Mixed NVLink transport, second pass (2 GPUs, config 3): every k-th remote operand staged by the
# copy engines, chunk count, first chunk folded straight from the peers.
OUT=${OUT:-gpurun_out/r02_hybrid2}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -k "staged" > $OUT/pytest_staged.log 2>&1; echo "rc=$?" >> $OUT/pytest_staged.log
run() {
  local name=$1; shift
  timeout 600 env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
     --master-port $((29900 + RANDOM % 500)) bench.py --gpus $NG --steps 10 --warmup 3 --no-e2e --no-variants \
     --no-cpu-baseline $BARGS > $OUT/$name.log 2>&1; echo rc=$? >> $OUT/$name.log
}
BARGS="--config 3 --mode fold" run fold_c3 MLF_X=0
for K in 2 3; do
  for CH in 4 8 16; do
    for FD in 0 1; do
      BARGS="--config 3 --mode staged" run e${K}_ch${CH}_fd${FD}_c3 MLF_STAGE_EVERY=$K MLF_STAGE_CHUNKS=$CH MLF_STAGE_FIRST_DIRECT=$FD
    done
  done
done
