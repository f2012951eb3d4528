mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py --n 8192 --steps 2 --warmup 3 --cpu-sample-s 15 > gpurun_out/bench_block.json 2> gpurun_out/bench_block.err; cat gpurun_out/bench_block.json; tail -3 gpurun_out/bench_block.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_block_n8192.csv python bench.py --n 8192 --steps 1 --warmup 0 --no-cpu --no-accuracy --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_gram|k_inner" -s 30 -c 3 -o gpurun_out/prof_block_n8192 python bench.py --n 8192 --steps 1 --warmup 0 --no-cpu --no-accuracy --e2e-steps 1 > gpurun_out/ncu_block.log 2>&1; tail -2 gpurun_out/ncu_block.log
