#!/bin/bash
# Multi-GPU evidence on one box: parity check, then bench at N = 2, 4, 8 (config 3) and config 5 at N = 8.
OUT=${OUT:-gpurun_out}
NG=$(nvidia-smi -L | wc -l)
timeout 300 python -m torch.distributed.run --standalone --nproc-per-node $NG tests/multigpu_check.py --cid 3 --S 4000037 > $OUT/check_n$NG.log 2>&1; echo rc=$? >> $OUT/check_n$NG.log
for N in 2 4 8; do
  [ $N -le $NG ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N \
     bench.py --gpus $N --steps 10 --warmup 3 > $OUT/bench_n$N.log 2>&1; echo rc=$? >> $OUT/bench_n$N.log
done
if [ $NG -ge 8 ]; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29599 \
     bench.py --gpus 8 --config 5 --steps 6 --warmup 3 --no-e2e > $OUT/bench_n8_cfg5.log 2>&1; echo rc=$? >> $OUT/bench_n8_cfg5.log
fi
# configs 4 (re-planned every batch, N2 NVLink shares, C2 stragglers) and 5 (replica, Div_max 0) at the largest N
NB=$([ $NG -ge 8 ] && echo 8 || echo $NG)
if [ $NB -ge 2 ]; then
  for C in 4 5; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NB --master-addr 127.0.0.1 --master-port 2957$C \
       bench.py --gpus $NB --config $C --steps 6 --warmup 3 --no-e2e --no-variants > $OUT/bench_n${NB}_cfg$C.log 2>&1; echo rc=$? >> $OUT/bench_n${NB}_cfg$C.log
  done
fi
