# round-2 checks: new GPU tests, the reference suite through the shim, the XL goldens, residual table
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_block.log 2>&1; tail -3 gpurun_out/pytest_block.log
timeout 1500 python -m pytest tests/test_gpu_reference_suite.py -q > gpurun_out/pytest_refsuite.log 2>&1; tail -3 gpurun_out/pytest_refsuite.log
timeout 900 python -m pytest tests/test_gpu_xl.py -q -s > gpurun_out/pytest_xl.log 2>&1; tail -8 gpurun_out/pytest_xl.log
timeout 900 python tools/block_residual_table.py > gpurun_out/residual_table.md 2>&1; tail -20 gpurun_out/residual_table.md
