#!/bin/bash
# Build an engine variant for tools/exp_variant.sh: bash tools/build_variant.sh NAME "-DFLAG=1 ..."
cd "$(dirname "$0")/.."
SRC="paper_2112_10239_b200/csrc/tq_engine.cu paper_2112_10239_b200/csrc/tq_trunc.cu"
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -cudart shared -Iinclude -diag-suppress 177,550"
nvcc $FLAGS $2 -Xptxas -v -o paper_2112_10239_b200/libtq_engine_$1.so $SRC > build_variant_$1.log 2>&1 &
P1=$!
nvcc $FLAGS $2 -DTQ_STAGE_TIMING -o paper_2112_10239_b200/libtq_engine_timing_$1.so $SRC > /dev/null 2>&1 &
P2=$!
wait $P1 || { tail -20 build_variant_$1.log; exit 1; }
wait $P2
echo built $1
