# inner rewrite check: block/sharded/xl GPU tests, one bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py tests/test_gpu_xl.py -q -x 2>&1 | tail -5
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-accuracy > gpurun_out/b_inner.json 2>gpurun_out/b_inner.err; python -c "
import json; d=json.loads(open('gpurun_out/b_inner.json').read().strip().splitlines()[-1]); print(d['value'], d['sweeps'], d['roofline']['kernel_ms_sweep0'], [round(x,1) for x in d['sweep_gpu_ms']])"
