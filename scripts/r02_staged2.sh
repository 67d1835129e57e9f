#!/bin/bash
# whole-slice staging (copy engines, one copy per remote operand slice) vs fold, N GPUs
OUT=${OUT:-gpurun_out/r02_staged}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x > $OUT/pytest_multirank_n$NG.log 2>&1; echo "rc=$?" >> $OUT/pytest_multirank_n$NG.log
for MODE in staged fold; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2962$NG \
     bench.py --gpus $NG --mode $MODE --steps 8 --warmup 3 --no-e2e --no-variants --no-cpu-baseline > $OUT/bench_n${NG}_$MODE.log 2>&1; echo rc=$? >> $OUT/bench_n${NG}_$MODE.log
done
MLF_STAGE_WHOLE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2963$NG \
   bench.py --gpus $NG --mode staged --steps 8 --warmup 3 --no-e2e --no-variants --no-cpu-baseline > $OUT/bench_n${NG}_staged_chunked.log 2>&1; echo rc=$? >> $OUT/bench_n${NG}_staged_chunked.log
for C in 4 5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2964$C \
     bench.py --gpus $NG --config $C --mode staged --steps 6 --warmup 3 --no-e2e --no-variants --no-cpu-baseline > $OUT/bench_n${NG}_cfg${C}_staged.log 2>&1; echo rc=$? >> $OUT/bench_n${NG}_cfg${C}_staged.log
done
