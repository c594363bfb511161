#!/bin/bash
# Round-2 GPU check: the GPU suite, the default bench line (cfg4) and the reference arm.
set -u
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/r2/bench_cfg4.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2/bench_cfg4.log | cut -c1-600
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2/ref_cfg4.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r2/ref_cfg4.log | cut -c1-400
