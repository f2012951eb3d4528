# ncu full capture of k_inner in the standalone bench (16 segments)
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k k_inner -s 3 -c 1 \
    -o gpurun_out/prof_inner_la tools/inner_bench 128 1 5 0 16 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
