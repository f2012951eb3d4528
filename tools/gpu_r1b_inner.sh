mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_block.py -x -q > gpurun_out/pytest_block.log 2>&1; tail -5 gpurun_out/pytest_block.log
for rot in fast dd; do
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --block-rotation $rot > gpurun_out/bench_$rot.json 2> gpurun_out/bench_$rot.err; cat gpurun_out/bench_$rot.json; tail -3 gpurun_out/bench_$rot.err
done
