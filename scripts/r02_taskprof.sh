#!/bin/bash
# Alg. 2 scan task profile on the GPU box's host (scripts/planbench/taskprof.cpp: items per scan,
# wall vs summed vs longest task per scan, per-thread task time) + planbench of the variants.
OUT=${OUT:-gpurun_out/r02_taskprof}
mkdir -p $OUT
python scripts/planbench/dump.py /tmp/planinst > $OUT/dump.log 2>&1
python scripts/planbench/taskprof.py > /tmp/planner_taskprof.cpp
g++ -O2 -std=c++17 -pthread -ffp-contract=off scripts/planbench/planbench.cpp /tmp/planner_taskprof.cpp -Iinclude -Ipaper_1907_00434_b200/csrc -o /tmp/pb_tp
for T in 1 2 4 8; do
  for ME in 2 4 8; do
    [ $T = 1 ] && [ $ME != 8 ] && continue
    echo "== threads $T min_evals $ME" >> $OUT/taskprof.log
    MLF_PLAN_MIN_EVALS=$ME MLF_PLAN_THREADS=$T /tmp/pb_tp /tmp/planinst/configs.txt 15 config4_G8 >> $OUT/taskprof.log 2>&1
  done
done
for V in paper_1907_00434_b200/csrc/planner.cpp; do
  n=$(basename $V .cpp)
  g++ -O2 -std=c++17 -pthread -ffp-contract=off scripts/planbench/planbench.cpp $V -Iinclude -Ipaper_1907_00434_b200/csrc -o /tmp/pb_$n
  for T in 1 4 8 16; do
    for ME in 4 8 32; do
      echo "== $n threads $T min_evals $ME" >> $OUT/planab.log
      MLF_PLAN_MIN_EVALS=$ME MLF_PLAN_THREADS=$T /tmp/pb_$n /tmp/planinst/configs.txt 15 >> $OUT/planab.log 2>&1
    done
  done
  MLF_PLAN_THREADS=8 MLF_PLAN_MIN_EVALS=2 /tmp/pb_$n /tmp/planinst/random.txt 1 | tail -1 >> $OUT/planab.log
done
