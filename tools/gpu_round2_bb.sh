# rotation c-from-t: inner latency, residual table, bench
mkdir -p gpurun_out
timeout 60 tools/inner_bench 128 1 20 0 16 2>&1 | grep 'k_inner<64>\|leader per round\|W^T' | head -3
timeout 1500 python tools/block_residual_table.py > gpurun_out/resid_table.md 2> gpurun_out/resid_table.err; tail -4 gpurun_out/resid_table.md
timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_bb.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_bb.json').read().strip().splitlines()[-1]); print(d['value'], d['sweeps'], d['clocks']['sm_mhz'], [round(x,1) for x in d['sweep_gpu_ms']])"
