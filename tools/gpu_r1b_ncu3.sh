mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update_p" -s 30 -c 1 -o gpurun_out/prof_updp python tools/block_sweep.py 8192 1 32 full > gpurun_out/ncu_updp.log 2>&1; tail -2 gpurun_out/ncu_updp.log
