mkdir -p gpurun_out
python tools/ab_variants.py "gmajor:" "qmajor:-DHSVD_GRAM_TMA_GMAJOR=0" \
  "k128s2o1:-DHSVD_GRAM_KT=128 -DHSVD_GRAM_STAGES=2 -DHSVD_GRAM_OCC=1 -DHSVD_GRAM_TMA_STAGES=2 -DHSVD_GRAM_TMA_OCC=1" \
  "k128s3o1:-DHSVD_GRAM_KT=128 -DHSVD_GRAM_STAGES=2 -DHSVD_GRAM_OCC=1 -DHSVD_GRAM_TMA_STAGES=3 -DHSVD_GRAM_TMA_OCC=1" \
  2>&1 | tee gpurun_out/ab_gram3.txt
HSVD_PLAN_STATS=1 python tools/block_telemetry.py 8192 2>&1 | grep -i "plan stats"
