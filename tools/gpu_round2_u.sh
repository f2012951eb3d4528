# ordering / passes A/B at n=8192 (sweeps and time)
mkdir -p gpurun_out
for args in "--inner-ordering full" "--inner-ordering oriented" "--inner-passes 2"; do
  timeout 600 python bench.py --steps 1 --warmup 2 --no-cpu $args > gpurun_out/b_u.json 2>/dev/null; python -c "
import json,sys; d=json.loads(open('gpurun_out/b_u.json').read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['sweeps'], d.get('accuracy'), [round(x,1) for x in d['sweep_gpu_ms']])" "$args"
done
