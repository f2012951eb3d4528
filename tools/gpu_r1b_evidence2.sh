mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 1500 gpurun_out/bench_default.json; tail -2 gpurun_out/bench_default.err
timeout 1200 python bench.py --mode pointwise --steps 1 --warmup 1 --no-cpu --no-accuracy > gpurun_out/bench_pointwise.json 2> gpurun_out/bench_pointwise.err; tail -c 600 gpurun_out/bench_pointwise.json; tail -2 gpurun_out/bench_pointwise.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; cat gpurun_out/bench_reference.json | tail -c 800
