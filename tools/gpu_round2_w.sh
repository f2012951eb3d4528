# block_streams 1 vs 2 with the rewritten inner
mkdir -p gpurun_out
for bs in 2 1 2 1; do
  timeout 600 python bench.py --steps 1 --warmup 2 --no-cpu --no-accuracy --block-streams $bs > gpurun_out/b_w.json 2>/dev/null; python -c "
import json,sys; d=json.loads(open('gpurun_out/b_w.json').read().strip().splitlines()[-1]); print('streams', sys.argv[1], d['value'], d['sweeps'], [round(x,1) for x in d['sweep_gpu_ms']])" $bs
done
