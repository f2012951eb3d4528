mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py --n 8192 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_block2.json 2> gpurun_out/bench_block2.err; cat gpurun_out/bench_block2.json; tail -3 gpurun_out/bench_block2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gram|k_inner" -s 20 -c 2 -o gpurun_out/prof_block2 python bench.py --n 8192 --steps 1 --warmup 0 --no-cpu --no-accuracy --e2e-steps 1 > gpurun_out/ncu_block2.log 2>&1; tail -1 gpurun_out/ncu_block2.log
