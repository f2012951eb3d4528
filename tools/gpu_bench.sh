# On a GPU box (gpurun): the contract bench lines (block default, pointwise,
# reference arm) into gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 1200 python bench.py --mode pointwise --steps 1 --warmup 1 --no-cpu --no-accuracy \
    > gpurun_out/bench_pointwise.json 2> gpurun_out/bench_pointwise.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 \
    > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
tail -c 400 gpurun_out/bench_default.json
