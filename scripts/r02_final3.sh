#!/bin/bash
# Round-2 final multi-GPU evidence (2 or 4 GPUs) on the round-end build: the 1-GPU parity file
# (the harness's batched push), the multi-rank GPU tests, bench at N GPUs with every variant,
# configs 4 and 5 at N GPUs.
OUT=${OUT:-gpurun_out/r02_final3}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu > $OUT/pytest_parity.log 2>&1; echo "rc=$?" >> $OUT/pytest_parity.log
timeout 1200 python -m pytest tests/test_gpu_multirank.py -q > $OUT/pytest_multirank_n$NG.log 2>&1; echo "rc=$?" >> $OUT/pytest_multirank_n$NG.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29801 \
   bench.py --gpus $NG --steps 10 --warmup 3 > $OUT/bench_n$NG.log 2>&1; echo rc=$? >> $OUT/bench_n$NG.log
for C in 4 5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2981$C \
     bench.py --gpus $NG --config $C --steps 6 --warmup 3 --no-e2e --no-variants > $OUT/bench_n${NG}_cfg$C.log 2>&1; echo rc=$? >> $OUT/bench_n${NG}_cfg$C.log
done
