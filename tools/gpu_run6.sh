mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py --n 8192 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_block3.json 2> gpurun_out/bench_block3.err; cat gpurun_out/bench_block3.json; tail -3 gpurun_out/bench_block3.err
