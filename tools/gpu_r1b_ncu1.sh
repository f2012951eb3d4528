mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_inner|k_update|k_gram" -s 30 -c 3 -o gpurun_out/prof_inner1 python tools/block_sweep.py 8192 1 > gpurun_out/ncu_inner1.log 2>&1; tail -3 gpurun_out/ncu_inner1.log
