for sg in 6 7 8 9 10 11; do
  python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --segments $sg > gpurun_out/seg_$sg.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/seg_$sg.log').read().strip().splitlines()[-1]);r=d['roofline'];print($sg, d['config'].get('sub_chain_sites'), round(d['value']), r['rl_ms'], r['lr_ms'], r['adj_ms'])"
done
