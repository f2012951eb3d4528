mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for n in 8192 4096; do for ps in 1 2 3; do
timeout 900 python bench.py --n $n --steps 1 --warmup 1 --no-cpu --inner-passes $ps 2> gpurun_out/bench_p.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['n'], d['config']['inner_passes'], round(d['value'],3), d['sweeps'], d['accuracy'], d['roofline']['kernel_ms_sweep0'], d['sweep_gpu_ms'])"
done; done
