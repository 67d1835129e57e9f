#!/bin/bash
# Single-thread and 8-thread planbench of the round-2 planner milestones (regression check).
OUT=${OUT:-gpurun_out/r02_planab1}
mkdir -p $OUT
python scripts/planbench/dump.py /tmp/planinst > $OUT/dump.log 2>&1
for V in scripts/planbench/variants/*.cpp; do
  n=$(basename $V .cpp)
  g++ -O2 -std=c++17 -pthread -ffp-contract=off scripts/planbench/planbench.cpp $V -Iinclude -Ipaper_1907_00434_b200/csrc -o /tmp/pb_$n 2>>$OUT/build.log
done
for rep in 1 2; do
for V in scripts/planbench/variants/*.cpp; do
  n=$(basename $V .cpp)
  for T in 1 8; do
    echo "== $n threads $T" >> $OUT/planab.log
    MLF_PLAN_MIN_EVALS=4 MLF_PLAN_THREADS=$T /tmp/pb_$n /tmp/planinst/configs.txt 15 >> $OUT/planab.log 2>&1
  done
done
done
