#!/bin/bash
# config 4 / config 3 at 4 GPUs: dynamic 1024-element tiles vs contiguous ranges (16 KB tiles)
OUT=${OUT:-gpurun_out/r02_contig4}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
for SC in dynamic contig; do
  for C in 4 3; do
    MLF_BULK_SCHED=$SC timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2961$C \
       bench.py --gpus $NG --config $C --steps 8 --warmup 3 --no-e2e --no-variants --no-cpu-baseline > $OUT/bench_n${NG}_cfg${C}_$SC.log 2>&1; echo rc=$? >> $OUT/bench_n${NG}_cfg${C}_$SC.log
  done
done
OUT=$OUT/planbox bash scripts/r02_planbox.sh
