set -u
bash tools/exp_variant.sh cfg4 "v0 t44" 2>&1
TQ_ENGINE_LIB=paper_2112_10239_b200/libtq_engine_t44.so timeout 900 python -m pytest tests/test_gpu_realpath.py tests/test_gpu_bench_plans.py tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -3
