# block/sharded/XL GPU tests (hang-safe) and one n=8192 bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py tests/test_gpu_xl.py -q -x --timeout=180 --timeout-method=thread > gpurun_out/pytest_s.log 2>&1
tail -3 gpurun_out/pytest_s.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-accuracy > gpurun_out/b_s.json 2>gpurun_out/b_s.err; python -c "
import json; d=json.loads(open('gpurun_out/b_s.json').read().strip().splitlines()[-1]); print(d['value'], d['sweeps'], d['roofline']['kernel_ms_sweep0'], d['clocks']['sm_mhz'], [round(x,1) for x in d['sweep_gpu_ms']])"
