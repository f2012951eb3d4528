# compact inner (co-resident with k_update) vs default: solve time A/B
mkdir -p gpurun_out
timeout 1500 python tools/ab_variants.py "default1:" "compact:-DHSVD_INNER_COMPACT=1" "default2:" "compact2:-DHSVD_INNER_COMPACT=1" > gpurun_out/ab_x.txt 2>/dev/null
grep -E '^(default|compact)' gpurun_out/ab_x.txt
