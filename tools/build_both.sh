#!/bin/bash
# Build the engine and its stage-timing variant in parallel (ptxas -v log in build_ptxas.log).
cd "$(dirname "$0")/.."
SRC="paper_2112_10239_b200/csrc/tq_engine.cu paper_2112_10239_b200/csrc/tq_trunc.cu"
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -cudart shared -Iinclude -diag-suppress 177,550"
nvcc $FLAGS -Xptxas -v -o paper_2112_10239_b200/libtq_engine.so.tmp $SRC > build_ptxas.log 2>&1 &
P1=$!
nvcc $FLAGS -DTQ_STAGE_TIMING -o paper_2112_10239_b200/libtq_engine_timing.so $SRC > build_timing.log 2>&1 &
P2=$!
wait $P1 || { tail -30 build_ptxas.log; exit 1; }
wait $P2 || { tail -30 build_timing.log; exit 1; }
mv paper_2112_10239_b200/libtq_engine.so.tmp paper_2112_10239_b200/libtq_engine.so
echo built
