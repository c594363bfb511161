#!/bin/bash
# Round-2 GPU check: precision diagnostic, the GPU suite, bench lines (cfg4 default, cfg2) and the reference arm.
set -u
mkdir -p gpurun_out/r2
timeout 300 python tools/prec_diag.py > gpurun_out/r2/prec.txt 2>&1; echo "prec rc=$?"; cat gpurun_out/r2/prec.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/r2/pytest_gpu.txt | tail -15
timeout 600 python bench.py > gpurun_out/r2/bench_cfg4.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2/bench_cfg4.log | cut -c1-300
timeout 600 python bench.py --config cfg2 > gpurun_out/r2/bench_cfg2.log 2>&1; echo "bench2 rc=$?"; tail -1 gpurun_out/r2/bench_cfg2.log | cut -c1-300
