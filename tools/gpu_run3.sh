mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_block.py -x -q 2>&1 | tail -25
timeout 600 python tools/block_check.py 2>&1 | tail -20
timeout 600 python bench.py --n 8192 --mode block --steps 1 --warmup 3 --no-cpu --e2e-steps 1 2>&1 | tail -3
