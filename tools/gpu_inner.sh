# k_inner A/B on a GPU box: standalone latency (k_inner vs v1 vs register
# kernel), one and 16 Gram segments per slot
mkdir -p gpurun_out
: > gpurun_out/inner_bench.txt
for args in "128 1 20 0 1" "128 1 20 0 16" "128 0 20 0 16" "128 1 20 1 16"; do
  echo "== inner_bench $args" >> gpurun_out/inner_bench.txt
  timeout 60 tools/inner_bench $args >> gpurun_out/inner_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/inner_bench.txt
done
cat gpurun_out/inner_bench.txt
