python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 4096 8192; do for bs in 2 1; do
timeout 300 python bench.py --n $n --steps 3 --warmup 2 --no-cpu --no-accuracy --block-streams $bs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['block_streams'], d['value'], d['sweeps'], d['host_phase_ms'], sum(d['sweep_gpu_ms']), d['sweep_gpu_ms'])"
done; done
