#!/bin/bash
# Race / uninitialised-read stress build (csrc/tq_debug.cuh): poisoned shared memory and
# randomly delayed barriers.  Loaded by tools/race_stress.py through TQ_ENGINE_LIB.
cd "$(dirname "$0")/.."
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -cudart shared \
  -Iinclude -diag-suppress 177,550 -DTQ_DEBUG_RACE -o paper_2112_10239_b200/libtq_engine_debug.so \
  paper_2112_10239_b200/csrc/tq_engine.cu paper_2112_10239_b200/csrc/tq_trunc.cu > build_debug.log 2>&1 \
  || { tail -30 build_debug.log; exit 1; }
echo built debug
