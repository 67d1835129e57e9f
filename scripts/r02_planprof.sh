#!/bin/bash
# Planner phase breakdown on the GPU box's host (scripts/planbench/prof.py timers) at 1-8 threads.
OUT=${OUT:-gpurun_out/r02_planprof}
mkdir -p $OUT
lscpu > $OUT/lscpu.txt
python scripts/planbench/dump.py /tmp/planinst > $OUT/dump.log 2>&1
python scripts/planbench/prof.py $PROF_ARGS > /tmp/planner_prof.cpp
g++ -O2 -std=c++17 -pthread -ffp-contract=off scripts/planbench/planbench.cpp /tmp/planner_prof.cpp -Iinclude -Ipaper_1907_00434_b200/csrc -o /tmp/pb_prof
for T in ${TS:-1 2 4 8 16}; do
  for ME in ${MES:-8 32}; do
    echo "== threads $T min_evals $ME" >> $OUT/prof.log
    MLF_PLAN_MIN_EVALS=$ME MLF_PLAN_THREADS=$T /tmp/pb_prof /tmp/planinst/configs.txt 15 config4_G8 >> $OUT/prof.log 2>&1
  done
done
