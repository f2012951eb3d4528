# late-sweep oriented ordering A/B: time, sweeps, XL residual gate
mkdir -p gpurun_out
for lo in 0 1; do
  HSVD_LATE_ORIENTED=$lo timeout 600 python bench.py --steps 1 --warmup 2 --no-cpu > gpurun_out/b_aa.json 2>/dev/null; python -c "
import json,sys; d=json.loads(open('gpurun_out/b_aa.json').read().strip().splitlines()[-1]); print('late oriented', sys.argv[1], d['value'], d['sweeps'], d.get('accuracy'), [round(x,1) for x in d['sweep_gpu_ms']])" $lo
  HSVD_LATE_ORIENTED=$lo timeout 900 python -m pytest tests/test_gpu_xl.py -q -s -k block --timeout=600 --timeout-method=thread 2>&1 | grep -E 'ratios|passed|failed'
done
