# ncu full capture of k_gram_tma (one-stream sweep, steps after warm-up) + source export
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_tma" \
    -s 20 -c 1 -o gpurun_out/prof_gram_tma python tools/block_sweep.py 8192 1 32 full 1 > gpurun_out/ncu_gram.log 2>&1
ncu -i gpurun_out/prof_gram_tma.ncu-rep --page raw --csv > gpurun_out/prof_gram_tma_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_gram_tma.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_gram_tma_src.csv 2>/dev/null
python tools/ncu_hot.py gpurun_out/prof_gram_tma_src.csv 30 > gpurun_out/prof_gram_tma_hot.txt 2>&1
head -60 gpurun_out/prof_gram_tma_hot.txt
