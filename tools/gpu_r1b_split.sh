mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_block.log 2>&1; tail -3 gpurun_out/pytest_block.log
for n in 8192 4096; do for bs in 2 1; do
timeout 300 python bench.py --n $n --steps 1 --warmup 1 --no-cpu --block-streams $bs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['n'], d['config']['block_streams'], d['value'], d['sweeps'], d['accuracy'], d['roofline']['kernel_ms_sweep0'], d['sweep_gpu_ms'][:3])"
done; done
