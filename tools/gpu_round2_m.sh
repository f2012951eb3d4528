mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
# sweep-0 (full class) and sweep-12 (cross class) Gram launches, tile TMA
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_tma" \
    -s 20 -c 1 -o gpurun_out/prof_gram_tile0 python tools/block_sweep.py 8192 1 32 full 1 > gpurun_out/ncu_g0.log 2>&1
HSVD_PROFILE_SWEEP=12 timeout 1200 ncu --set full --clock-control none -k regex:"k_gram_tma" \
    -s 3090 -c 1 -o gpurun_out/prof_gram_tile12 python tools/profile_sweep.py 8192 > gpurun_out/ncu_g12.log 2>&1
for f in prof_gram_tile0 prof_gram_tile12; do
ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
done
ncu -i gpurun_out/prof_gram_tile0.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_gram_tile0_src.csv 2>/dev/null
python tools/ncu_hot.py gpurun_out/prof_gram_tile0_src.csv 12 | head -30
tail -3 gpurun_out/ncu_g12.log
