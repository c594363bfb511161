#!/bin/bash
mkdir -p gpurun_out/st
timeout 1200 python -m pytest tests/test_gpu_states.py tests/test_gpu_trunc.py tests/test_gpu_cli.py tests/test_gpu_api.py -q --timeout 900 > gpurun_out/st/pytest.txt 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error|^E  " gpurun_out/st/pytest.txt | tail -25
