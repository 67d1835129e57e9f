#!/bin/bash
OUT=${OUT:-gpurun_out/r02_staged3}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
for SS in 1 2 4; do
  for GG in 4 8 16; do
    MLF_STAGE_STREAMS=$SS MLF_STAGE_GROUPS=$GG timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 297$SS$GG \
       bench.py --gpus $NG --mode staged --steps 6 --warmup 2 --no-e2e --no-variants --no-cpu-baseline > $OUT/bench_n${NG}_staged_s${SS}_g$GG.log 2>&1
  done
done
