#!/bin/bash
# Round-end multi-GPU check on the final build: multi-rank GPU tests, the default N-GPU bench line
# (every variant, the mixed transport at 3 of 4 operands staged), config 4.
OUT=${OUT:-gpurun_out/r02_final12}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_gpu_multirank.py -q > $OUT/pytest_multirank_n$NG.log 2>&1; echo "rc=$?" >> $OUT/pytest_multirank_n$NG.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29811 \
   bench.py --gpus $NG --steps 10 --warmup 3 > $OUT/bench_n$NG.log 2>&1; echo rc=$? >> $OUT/bench_n$NG.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29814 \
   bench.py --gpus $NG --config 4 --steps 6 --warmup 3 --no-e2e --no-variants > $OUT/bench_n${NG}_cfg4.log 2>&1; echo rc=$? >> $OUT/bench_n${NG}_cfg4.log
