# inner passes with the accurate rotation: time, sweeps, XL gate, residual table
mkdir -p gpurun_out
for cfg in "P1::" "P2:--inner-passes 2:" "D2::2"; do
  name=${cfg%%:*}; rest=${cfg#*:}; args=${rest%%:*}; dp=${rest#*:}
  HSVD_DENSE_PASSES=${dp:-1} timeout 600 python bench.py --steps 1 --warmup 2 --no-cpu --no-accuracy $args > gpurun_out/b_ff.json 2>/dev/null; python -c "
import json,sys; d=json.loads(open('gpurun_out/b_ff.json').read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['sweeps'], d['clocks']['sm_mhz'], [round(x,1) for x in d['sweep_gpu_ms']])" $name
done
HSVD_DENSE_PASSES=2 timeout 900 python -m pytest tests/test_gpu_xl.py -q -s -k block --timeout=600 --timeout-method=thread 2>&1 | grep -E 'ratios|passed|failed'
