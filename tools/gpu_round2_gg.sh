# dense passes 3 vs auto (2) with the accurate rotation: time, sweeps, XL gate
mkdir -p gpurun_out
for dp in 2 3; do
  HSVD_DENSE_PASSES=$dp timeout 600 python bench.py --steps 1 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_gg.json 2>/dev/null; python -c "
import json,sys; d=json.loads(open('gpurun_out/b_gg.json').read().strip().splitlines()[-1]); print('dense passes', sys.argv[1], d['value'], d['sweeps'], d['clocks']['sm_mhz'], [round(x,1) for x in d['sweep_gpu_ms']])" $dp
  HSVD_DENSE_PASSES=$dp timeout 900 python -m pytest tests/test_gpu_xl.py -q -s -k block --timeout=600 --timeout-method=thread 2>&1 | grep -E 'ratios|passed|failed'
done
