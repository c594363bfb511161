set -u
bash tools/exp_variant.sh cfg4 "t44 f4" 2>&1
bash tools/exp_variant.sh cfg2 "v0 f4" 2>&1 | grep -v "cyc"
TQ_ENGINE_LIB=paper_2112_10239_b200/libtq_engine_f4.so timeout 900 python -m pytest tests/test_gpu_realpath.py tests/test_gpu_bench_plans.py tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -3
