# fast math accuracy, inner latency, residual table
mkdir -p gpurun_out
tools/rsqrt_acc
timeout 60 tools/inner_bench 128 1 20 0 16 2>&1 | grep 'k_inner<64>\|leader per round' | head -2
timeout 1500 python tools/block_residual_table.py > gpurun_out/resid_table.md 2> gpurun_out/resid_table.err; tail -1 gpurun_out/resid_table.md
