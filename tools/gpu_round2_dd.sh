# default c-from-t rotation: block/sharded/XL tests, residual table, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py tests/test_gpu_xl.py -q -x --timeout=300 --timeout-method=thread > gpurun_out/pytest_dd.log 2>&1; tail -2 gpurun_out/pytest_dd.log
timeout 1500 python tools/block_residual_table.py > gpurun_out/resid_table.md 2> gpurun_out/resid_table.err; tail -2 gpurun_out/resid_table.md
for i in 1 2; do timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_dd.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_dd.json').read().strip().splitlines()[-1]); print(d['value'], d['sweeps'], d['clocks']['sm_mhz'], [round(x,1) for x in d['sweep_gpu_ms']])"; done
