set -u
mkdir -p gpurun_out/ev2
timeout 900 bash tools/race_check.sh > gpurun_out/ev2/race.txt 2>&1; echo "race rc=$?"; tail -3 gpurun_out/ev2/race.txt
for c in cfg4 cfg2 cfg1 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/ev2/bench_$c.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/ev2/bench_$c.log > gpurun_out/ev2/bench_$c.json
done
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/ev2/bench_default.log 2>&1; echo "default rc=$?"
tail -1 gpurun_out/ev2/bench_default.log
