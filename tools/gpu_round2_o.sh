python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/gram_floor.py; HSVD_PROFILE_SWEEP=12 python tools/profile_sweep.py 8192 | grep kernel
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -2
timeout 400 python bench.py --steps 2 --warmup 3 --no-cpu --no-accuracy > gpurun_out/b_role.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_role.json').read().strip().splitlines()[-1]); print(d['value'], d['sweeps'], d['roofline']['kernel_ms_sweep0'], [round(x,1) for x in d['sweep_gpu_ms']])"
