mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for n in 8192 4096; do
timeout 900 python bench.py --n $n --steps 1 --warmup 1 --no-cpu --inner-ordering full 2> gpurun_out/bench_full.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['n'], d['value'], d['sweeps'], d['accuracy'], d['sweep_gpu_ms'])"
timeout 900 python bench.py --n $n --steps 1 --warmup 1 --no-cpu 2> gpurun_out/bench_or.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['n'], d['value'], d['sweeps'], d['accuracy'], d['sweep_gpu_ms'])"
done
