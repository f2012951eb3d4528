mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b1.json 2> gpurun_out/b1.err
tail -c 1500 gpurun_out/b1.json
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -30 gpurun_out/pytest_gpu.log
