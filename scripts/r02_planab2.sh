#!/bin/bash
# Planner A/B on the box host at 8 and 16 threads (variants in scripts/planbench/variants/).
OUT=${OUT:-gpurun_out/r02_planab2}
mkdir -p $OUT
nproc > $OUT/host.txt
python scripts/planbench/dump.py /tmp/planinst > $OUT/dump.log 2>&1
for V in scripts/planbench/variants/*.cpp; do
  n=$(basename $V .cpp)
  g++ -O2 -std=c++17 -pthread -ffp-contract=off scripts/planbench/planbench.cpp $V -Iinclude -Ipaper_1907_00434_b200/csrc -o /tmp/pb_$n 2>>$OUT/build.log
done
for rep in 1 2; do
for V in scripts/planbench/variants/*.cpp; do
  n=$(basename $V .cpp)
  for T in ${THREADS:-8 16}; do
    echo "== $n threads $T rep $rep" >> $OUT/planab.log
    MLF_PLAN_THREADS=$T /tmp/pb_$n /tmp/planinst/configs.txt 15 >> $OUT/planab.log 2>&1
  done
done
done
