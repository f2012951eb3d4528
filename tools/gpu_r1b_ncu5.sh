python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pointwise_stream" -s 20 -c 1 -o gpurun_out/prof_pw python tools/ncu_pointwise.py 8192 > gpurun_out/ncu_pw.log 2>&1; tail -1 gpurun_out/ncu_pw.log
