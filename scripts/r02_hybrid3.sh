#!/bin/bash
# Mixed NVLink transport, third pass (configs 3 and 5, fewer chunks with the first chunk direct),
# then the planner A/B of the current variants.
OUT=${OUT:-gpurun_out/r02_hybrid3}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
run() {
  local name=$1; shift
  timeout 600 env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
     --master-port $((29900 + RANDOM % 500)) bench.py --gpus $NG --steps 10 --warmup 3 --no-e2e --no-variants \
     --no-cpu-baseline $BARGS > $OUT/$name.log 2>&1; echo rc=$? >> $OUT/$name.log
}
for CH in 2 3 4; do
  BARGS="--config 3 --mode staged" run e2_ch${CH}_fd1_c3 MLF_STAGE_EVERY=2 MLF_STAGE_CHUNKS=$CH MLF_STAGE_FIRST_DIRECT=1
done
BARGS="--config 5 --mode fold --steps 6" run fold_c5 MLF_X=0
BARGS="--config 5 --mode staged --steps 6" run e2_ch4_fd1_c5 MLF_STAGE_EVERY=2 MLF_STAGE_CHUNKS=4 MLF_STAGE_FIRST_DIRECT=1
OUT=gpurun_out/r02_planab MES=4 bash scripts/r02_planab.sh
