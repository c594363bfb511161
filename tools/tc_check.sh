timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_api.py -q -x 2>&1 | tail -2
for tc in 1 0; do
  TQ_TC=$tc timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_tc$tc.log 2>&1
  tail -1 gpurun_out/b4_tc$tc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('TC', $tc, round(d['value'],1), r['rl_ms'], r['lr_ms'], r['adj_ms'])" 2>&1 | tail -1
done
