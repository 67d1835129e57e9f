#!/bin/bash
OUT=${OUT:-gpurun_out/r02_c6}
mkdir -p $OUT
OUT=$OUT/planbox bash scripts/r02_planbox.sh
timeout 600 python -m torch.distributed.run --standalone --nnodes=1 --nproc-per-node=2 tests/multigpu_check.py --cid 5 --S 200003 --steps 4 --replica-mode 1 --div-max 20 --workers 32 --modes fold,tree,staged > $OUT/mgcheck_cid5.log 2>&1; echo "rc=$?" >> $OUT/mgcheck_cid5.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_default.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
