# On a GPU box (gpurun): everything the round's evidence needs, in one call:
# GPU tests, the contract bench lines, the ncu launch list of one sweep and
# full captures of the block kernels (one-stream step) and of the pointwise
# step kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout=600 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1
tail -12 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -c 400 gpurun_out/bench_default.json
timeout 1200 python bench.py --mode pointwise --steps 1 --warmup 3 --no-cpu --no-accuracy \
    > gpurun_out/bench_pointwise.json 2> gpurun_out/bench_pointwise.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 \
    > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file gpurun_out/launches_block.csv python tools/block_sweep.py 8192 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_gram|k_inner" \
    -s 40 -c 3 -o gpurun_out/prof_block python tools/block_sweep.py 8192 1 32 full 1 > /dev/null 2>&1
ncu -i gpurun_out/prof_block.ncu-rep --page raw --csv > gpurun_out/prof_block_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pointwise_stream" \
    -s 20 -c 1 -o gpurun_out/prof_pointwise python tools/ncu_pointwise.py 8192 > /dev/null 2>&1
ncu -i gpurun_out/prof_pointwise.ncu-rep --page raw --csv > gpurun_out/prof_pointwise_raw.csv 2>/dev/null
ls gpurun_out | head -60
