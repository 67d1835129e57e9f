#!/bin/bash
# Planner A/B on the box host: variants x helper-thread counts at 8 planner threads.
OUT=${OUT:-gpurun_out/r02_planab3}
mkdir -p $OUT
nproc > $OUT/host.txt
python scripts/planbench/dump.py /tmp/planinst > $OUT/dump.log 2>&1
for V in scripts/planbench/variants/*.cpp; do
  n=$(basename $V .cpp)
  g++ -O2 -std=c++17 -pthread -ffp-contract=off scripts/planbench/planbench.cpp $V -Iinclude -Ipaper_1907_00434_b200/csrc -o /tmp/pb_$n 2>>$OUT/build.log
done
for rep in ${REPS:-1 2}; do
for V in scripts/planbench/variants/*.cpp; do
  n=$(basename $V .cpp)
  for H in ${HELPERS:-0 1 2 4}; do
    for T in ${THREADS:-8}; do
      echo "== $n helpers $H threads $T rep $rep" >> $OUT/planab.log
      MLF_PLAN_HELPERS=$H MLF_PLAN_THREADS=$T /tmp/pb_$n /tmp/planinst/configs.txt 15 config >> $OUT/planab.log 2>&1
    done
  done
done
done
