#!/bin/bash
# Batched submit: its GPU tests, then the bench line (variants off) for the device-resident leg.
OUT=${OUT:-gpurun_out/r02_devres}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_c_abi.py -q -m gpu -k "submit_batch or c99 or delay_bound or invalid_plan" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-variants --no-cpu-baseline > $OUT/bench.log 2>&1; echo "rc=$?" >> $OUT/bench.log
