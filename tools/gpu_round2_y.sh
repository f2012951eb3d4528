# pointwise variants A/B: sweeps 0-1 at n=8192 per variant
mkdir -p gpurun_out
AB_SCRIPT="tools/pw_sweep0.py 8192" timeout 1500 python tools/ab_variants.py "s16vb16:-DHSVD_PW_VBATCH=16" "s16vb12:-DHSVD_PW_VBATCH=12" "s16vb10:-DHSVD_PW_VBATCH=10" > gpurun_out/ab_y.txt 2>/dev/null
grep -E '^s' gpurun_out/ab_y.txt
