# On a GPU box (gpurun): ncu launch list of one block sweep and full captures
# of the block kernels (one-stream step) and of the pointwise step kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
    --log-file gpurun_out/launches_block.csv python tools/block_sweep.py 8192 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_gram|k_inner" \
    -s 40 -c 3 -o gpurun_out/prof_block python tools/block_sweep.py 8192 1 32 full 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pointwise_stream" \
    -s 20 -c 1 -o gpurun_out/prof_pointwise python tools/ncu_pointwise.py 8192 > /dev/null 2>&1
ls gpurun_out
