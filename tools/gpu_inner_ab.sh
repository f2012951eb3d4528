# k_inner variants side by side (tools/inner_bench_* builds)
mkdir -p gpurun_out
: > gpurun_out/inner_ab.txt
for b in tools/inner_bench tools/inner_bench_*; do
  [ -x $b ] || continue
  echo "== $b" >> gpurun_out/inner_ab.txt
  timeout 60 $b 128 1 20 0 16 2>&1 | grep 'k_inner<64>\|leader\|bulk\|prologue\|W^T' | head -6 >> gpurun_out/inner_ab.txt
done
cat gpurun_out/inner_ab.txt
