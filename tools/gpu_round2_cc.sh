# c from t (library rsqrt): inner latency and residual table
mkdir -p gpurun_out
timeout 60 tools/inner_bench_ct 128 1 20 0 16 2>&1 | grep 'k_inner<64>\|leader per round' | head -2
AB_SCRIPT="tools/block_residual_table.py" timeout 2000 python tools/ab_variants.py "ct:-DHSVD_ROT_C_FROM_T=1" > gpurun_out/ab_cc.txt 2>/dev/null
grep -E '^ct' gpurun_out/ab_cc.txt
