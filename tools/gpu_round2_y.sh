# pointwise V-batch A/B: sweeps 0-1 at n=8192 per variant
mkdir -p gpurun_out
AB_SCRIPT="tools/pw_sweep0.py 8192" timeout 1500 python tools/ab_variants.py "vb1:-DHSVD_PW_VBATCH=1" "vb4:-DHSVD_PW_VBATCH=4" "vb8:-DHSVD_PW_VBATCH=8" > gpurun_out/ab_y.txt 2>/dev/null
grep -E '^vb' gpurun_out/ab_y.txt
