# Round-1 evidence run: tests, smoke, default bench, ncu launch list + full captures.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json; tail -2 gpurun_out/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_block.csv python tools/block_sweep.py 8192 1 > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_gram|k_inner" -s 60 -c 3 -o gpurun_out/prof_block_full python tools/block_sweep.py 8192 1 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
