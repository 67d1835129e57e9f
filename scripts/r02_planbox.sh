#!/bin/bash
# Planner timing on the GPU box's host: planbench (C++ replay of dumped instances, per-instance
# best of 15) single-threaded and with 2/4/8 threads, and the instrumented phase breakdown.
OUT=${OUT:-gpurun_out/r02_planbox}
mkdir -p $OUT
python scripts/planbench/dump.py /tmp/planinst > $OUT/dump.log 2>&1
g++ -O2 -std=c++17 -pthread -ffp-contract=off scripts/planbench/planbench.cpp paper_1907_00434_b200/csrc/planner.cpp -Iinclude -o /tmp/planbench
for T in 1 2 4 8; do
  echo "== threads $T" >> $OUT/planbench.log
  MLF_PLAN_THREADS=$T /tmp/planbench /tmp/planinst/configs.txt 15 >> $OUT/planbench.log 2>&1
done
MLF_PLAN_THREADS=1 /tmp/planbench /tmp/planinst/random.txt 1 | tail -1 >> $OUT/planbench.log
for ME in 16 32 48; do
  for T in 4 8; do
    echo "== threads $T min_evals $ME" >> $OUT/planbench.log
    MLF_PLAN_MIN_EVALS=$ME MLF_PLAN_THREADS=$T /tmp/planbench /tmp/planinst/configs.txt 15 config4_G8 >> $OUT/planbench.log 2>&1
    MLF_PLAN_MIN_EVALS=$ME MLF_PLAN_THREADS=$T /tmp/planbench /tmp/planinst/configs.txt 15 config5 >> $OUT/planbench.log 2>&1
  done
done
if [ -f scripts/planbench/prof.py ]; then
  python scripts/planbench/prof.py > /tmp/planner_prof.cpp && g++ -O2 -std=c++17 -pthread -ffp-contract=off scripts/planbench/planbench.cpp /tmp/planner_prof.cpp -Iinclude -Ipaper_1907_00434_b200/csrc -o /tmp/planbench_prof
  for c in config4_G8 config5 config3_G8 config2_G1_tau32; do
    echo "== $c" >> $OUT/phases.log
    MLF_PLAN_THREADS=1 /tmp/planbench_prof /tmp/planinst/configs.txt 15 $c >> $OUT/phases.log 2>&1
  done
fi
