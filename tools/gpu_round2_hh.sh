# dense-sweep threshold for the 2-pass policy: 1/20 (default) vs 1/100 vs 1/1000
mkdir -p gpurun_out
for dv in 20 100 1000; do
  HSVD_DENSE_DIV=$dv timeout 600 python bench.py --steps 1 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_hh.json 2>/dev/null; python -c "
import json,sys; d=json.loads(open('gpurun_out/b_hh.json').read().strip().splitlines()[-1]); print('div', sys.argv[1], d['value'], d['sweeps'], d['clocks']['sm_mhz'], [round(x,1) for x in d['sweep_gpu_ms']])" $dv
  HSVD_DENSE_DIV=$dv timeout 900 python -m pytest tests/test_gpu_xl.py -q -s -k block --timeout=600 --timeout-method=thread 2>&1 | grep -E 'n8192.*ratios|passed|failed'
done
