set -u
bash tools/exp_variant.sh cfg4 "f4 h4" 2>&1
TQ_ENGINE_LIB=paper_2112_10239_b200/libtq_engine_h4.so timeout 900 python -m pytest tests/test_gpu_realpath.py tests/test_gpu_bench_plans.py tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -3
grep -A8 "^LR" gpurun_out/st_h4.txt
