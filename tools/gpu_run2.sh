set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
./tools/fp64_micro > gpurun_out/fp64_micro.json 2>&1; cat gpurun_out/fp64_micro.json
timeout 900 python bench.py --n 8192 --steps 1 --warmup 3 --cpu-sample-s 20 > gpurun_out/bench_n8192_pointwise.json 2> gpurun_out/bench_n8192.err; cat gpurun_out/bench_n8192_pointwise.json; tail -3 gpurun_out/bench_n8192.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pointwise_step -s 200 -c 2 -o gpurun_out/prof_pointwise_n8192 python tools/ncu_pointwise.py 8192 > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 400 --csv --log-file gpurun_out/launches_n8192.csv python tools/ncu_pointwise.py 8192 > /dev/null 2>&1
