#!/bin/bash
# ncu evidence for the 1-GPU bench line (run under gpurun, one GPU).
# 1) plain run must exit 0; 2) launch list (every kernel's device time, cold, serialised);
# 3) one --set full capture of the dominant kernel.
set -u
OUT=${OUT:-gpurun_out}
ARGS=${ARGS:-"--steps 3 --warmup 2 --no-variants --no-e2e --no-cpu-baseline"}
mkdir -p $OUT
python bench.py $ARGS > $OUT/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py $ARGS > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?" >> $OUT/prof_plain.log
python bench.py $ARGS > $OUT/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-fused_commit} -s ${SKIP:-2} -c ${COUNT:-2} \
    -o $OUT/prof_commit -f python bench.py $ARGS > $OUT/ncu_full.log 2>&1
echo "full rc=$?" >> $OUT/prof_plain.log
