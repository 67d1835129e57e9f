#!/bin/bash
# Mixed NVLink transport A/B (2 GPUs): staged mode with only every k-th remote operand pulled by
# the copy engines (MLF_STAGE_EVERY=k), the rest SM peer loads; fold as the baseline.
OUT=${OUT:-gpurun_out/r02_hybrid}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -k "staged" > $OUT/pytest_staged.log 2>&1; echo "rc=$?" >> $OUT/pytest_staged.log
run() {  # name, env..., -- bench args
  local name=$1; shift
  timeout 600 env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
     --master-port $((29900 + RANDOM % 500)) bench.py --gpus $NG --steps 10 --warmup 3 --no-e2e --no-variants \
     --no-cpu-baseline $BARGS > $OUT/$name.log 2>&1; echo rc=$? >> $OUT/$name.log
}
for C in 3 4; do
  BARGS="--config $C --mode fold" run fold_c$C MLF_X=0
  for K in 1 2 3 4 6; do
    BARGS="--config $C --mode staged" run staged_every${K}_c$C MLF_STAGE_EVERY=$K
  done
done
