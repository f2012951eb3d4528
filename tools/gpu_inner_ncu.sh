# ncu full capture of k_inner (new) and k_inner_v1 in the standalone bench
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_inner" -s 3 -c 1 \
    -o gpurun_out/prof_inner_new tools/inner_bench 128 1 5 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_inner_v1" -s 3 -c 1 \
    -o gpurun_out/prof_inner_v1 tools/inner_bench 128 1 5 0 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
