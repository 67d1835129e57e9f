#!/bin/bash
OUT=${OUT:-gpurun_out/r02_c5}
mkdir -p $OUT
timeout 600 python -m torch.distributed.run --standalone --nnodes=1 --nproc-per-node=2 tests/multigpu_check.py --cid 5 --S 200003 --steps 4 --replica-mode 1 --div-max 20 --workers 32 --modes fold,tree,staged > $OUT/mgcheck_cid5.log 2>&1; echo "rc=$?" >> $OUT/mgcheck_cid5.log
bash scripts/r02_planbox.sh
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
