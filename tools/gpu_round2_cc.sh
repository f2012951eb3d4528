# library sqrt/rsqrt/div in the fast rotation: inner latency and residual table
mkdir -p gpurun_out
timeout 60 tools/inner_bench_libm 128 1 20 0 16 2>&1 | grep 'k_inner<64>\|leader per round' | head -2
AB_SCRIPT="tools/block_residual_table.py" timeout 2000 python tools/ab_variants.py "libm:-DHSVD_ROT_LIBM=1" > gpurun_out/ab_cc.txt 2>/dev/null
grep -E '^libm' gpurun_out/ab_cc.txt
