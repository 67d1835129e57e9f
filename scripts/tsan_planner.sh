#!/bin/bash
# The host planner's thread pool under ThreadSanitizer, driven by the differential
# planner tests (C++ plan == oracle plan).  Host only (no GPU work is launched).
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1907_00434_b200/build
make -C paper_1907_00434_b200/csrc > /dev/null      # the (uninstrumented) CUDA objects
g++ -O1 -g -fsanitize=thread -fno-omit-frame-pointer -std=c++17 \
    -ffp-contract=off -pthread -fPIC -shared -Iinclude -Ipaper_1907_00434_b200/csrc -I/usr/local/cuda/include \
    paper_1907_00434_b200/csrc/planner.cpp paper_1907_00434_b200/csrc/executor.cpp \
    paper_1907_00434_b200/build/commit.o paper_1907_00434_b200/build/bulk.o paper_1907_00434_b200/build/synth.o \
    -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -o paper_1907_00434_b200/build/libmlfplan_tsan.so
TSAN_LIB=$(g++ -print-file-name=libtsan.so)
MLF_LIB=$PWD/paper_1907_00434_b200/build/libmlfplan_tsan.so LD_PRELOAD="$TSAN_LIB" \
TSAN_OPTIONS="halt_on_error=1 report_signal_unsafe=0" python -m pytest tests/test_planner_parity.py \
    tests/test_planner_distribution_parity.py -q -x -k "larger or 64 or box or degraded" -p no:cacheprovider
# the NEXT-2 Div_max stream (32 classes per scan, replica plans, carried items) with every Alg. 2
# scan on the pool: the case that exposed a late claim running an item of the next job
MLF_LIB=$PWD/paper_1907_00434_b200/build/libmlfplan_tsan.so LD_PRELOAD="$TSAN_LIB" MLF_PLAN_THREADS=8 MLF_PLAN_MIN_EVALS=2 \
TSAN_OPTIONS="halt_on_error=1 report_signal_unsafe=0" python -m pytest tests/test_replica_divmax_trend.py -q -x \
    -p no:cacheprovider
