#!/bin/bash
# Planner A/B on the GPU box's host: each scripts/planbench/variants/*.cpp (a planner.cpp variant)
# replayed by planbench at several thread counts and scan thresholds; plans must match.
OUT=${OUT:-gpurun_out/r02_planab}
mkdir -p $OUT
nproc > $OUT/host.txt; lscpu | head -20 >> $OUT/host.txt
python scripts/planbench/dump.py /tmp/planinst > $OUT/dump.log 2>&1
for V in scripts/planbench/variants/*.cpp; do
  n=$(basename $V .cpp)
  g++ -O2 -std=c++17 -pthread -ffp-contract=off scripts/planbench/planbench.cpp $V -Iinclude -Ipaper_1907_00434_b200/csrc -o /tmp/pb_$n 2>>$OUT/build.log || continue
done
for V in scripts/planbench/variants/*.cpp; do
  n=$(basename $V .cpp)
  for T in 1 4 8; do
    for ME in ${MES:-8 16 32}; do
      [ $T = 1 ] && [ $ME != 32 ] && continue
      echo "== $n threads $T min_evals $ME" >> $OUT/planab.log
      MLF_PLAN_MIN_EVALS=$ME MLF_PLAN_THREADS=$T /tmp/pb_$n /tmp/planinst/configs.txt 15 >> $OUT/planab.log 2>&1
    done
  done
  MLF_PLAN_THREADS=4 MLF_PLAN_MIN_EVALS=8 /tmp/pb_$n /tmp/planinst/random.txt 1 | tail -1 >> $OUT/planab.log
done
