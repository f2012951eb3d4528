mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_block.log 2>&1; tail -3 gpurun_out/pytest_block.log
python tools/block_telemetry.py 8192
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; cat gpurun_out/bench_n1.json; tail -3 gpurun_out/bench_n1.err
