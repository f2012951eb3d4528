python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_block.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 1 --warmup 2 --no-cpu --no-accuracy --sharded 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sharded N=1', round(d['value'],4), d['sweeps'], d['sweep_gpu_ms'][:3])"
