# k_inner A/B on a GPU box: standalone latency (new vs v1 vs register kernel)
# and the diagnostic variants (no W replay / no block updates)
mkdir -p gpurun_out
: > gpurun_out/inner_bench.txt
for b in inner_bench inner_bench_dnow1 inner_bench_dnoupd1; do
  [ -x tools/$b ] || continue
  echo "== $b 128 1 20 0" >> gpurun_out/inner_bench.txt
  if [ $b = inner_bench ]; then n=100; else n=4; fi
  timeout 60 tools/$b 128 1 20 0 2>&1 | head -$n >> gpurun_out/inner_bench.txt; echo "rc=$?" >> gpurun_out/inner_bench.txt
done
cat gpurun_out/inner_bench.txt
