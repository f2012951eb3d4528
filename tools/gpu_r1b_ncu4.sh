mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_gram" -s 40 -c 2 -o gpurun_out/prof_single python tools/block_sweep.py 8192 1 32 full 1 > gpurun_out/ncu_single.log 2>&1; tail -1 gpurun_out/ncu_single.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_single.csv python tools/block_sweep.py 8192 1 32 full 1 > /dev/null 2>&1
