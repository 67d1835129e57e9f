#!/bin/bash
# The host planner under AddressSanitizer + UndefinedBehaviorSanitizer, driven by the
# differential instances (C++ plan == oracle plan) of tests/test_planner_parity.py.
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1907_00434_b200/build
make -C paper_1907_00434_b200/csrc > /dev/null      # the (uninstrumented) CUDA objects
g++ -O1 -g -fsanitize=address,undefined -fno-sanitize-recover=undefined -fno-omit-frame-pointer -std=c++17 \
    -ffp-contract=off -pthread -fPIC -shared -Iinclude -Ipaper_1907_00434_b200/csrc -I/usr/local/cuda/include \
    paper_1907_00434_b200/csrc/planner.cpp paper_1907_00434_b200/csrc/executor.cpp \
    paper_1907_00434_b200/build/commit.o paper_1907_00434_b200/build/bulk.o paper_1907_00434_b200/build/synth.o \
    -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -o paper_1907_00434_b200/build/libmlfplan_asan.so
ASAN_LIB=$(g++ -print-file-name=libasan.so)
UBSAN_LIB=$(g++ -print-file-name=libubsan.so)
MLF_LIB=$PWD/paper_1907_00434_b200/build/libmlfplan_asan.so LD_PRELOAD="$ASAN_LIB $UBSAN_LIB" \
ASAN_OPTIONS=detect_leaks=0 python -m pytest tests/test_planner_parity.py -q -x -k "random or larger or paper or errors" -p no:cacheprovider
