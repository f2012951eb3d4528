python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 8192 4096; do
timeout 300 python bench.py --n $n --steps 2 --warmup 2 --no-cpu --no-accuracy 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['n'], round(d['value'],4), d['sweeps'], d['roofline']['kernel_ms_sweep0'], d['sweep_gpu_ms'][:2])"
done
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -1
