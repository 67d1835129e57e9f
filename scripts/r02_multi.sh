#!/bin/bash
# Round-2 multi-GPU evidence on one box (2 or 4 GPUs): multi-rank GPU tests, bench at N GPUs
# (rank-0 planning, cpu_baseline, same workload on one GPU), the bidirectional NVLink probe.
OUT=${OUT:-gpurun_out/r02_multi}
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
echo "gpus=$NG" > $OUT/info.txt
nvidia-smi topo -m >> $OUT/info.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -q > $OUT/pytest_multirank_n$NG.log 2>&1; echo "rc=$?" >> $OUT/pytest_multirank_n$NG.log
timeout 300 python scripts/nvlink_bidir_probe.py > $OUT/nvlink_bidir_probe.log 2>&1
for N in 2 4; do
  [ $N -le $NG ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N \
     bench.py --gpus $N --steps 10 --warmup 3 > $OUT/bench_n$N.log 2>&1; echo rc=$? >> $OUT/bench_n$N.log
done
NB=$NG
for C in 4 5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NB --master-addr 127.0.0.1 --master-port 2957$C \
     bench.py --gpus $NB --config $C --steps 6 --warmup 3 --no-e2e --no-variants > $OUT/bench_n${NB}_cfg$C.log 2>&1; echo rc=$? >> $OUT/bench_n${NB}_cfg$C.log
done
