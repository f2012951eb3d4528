set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 300 python tools/fp64_peak.py 8192 > gpurun_out/fp64_peak.json 2>&1; cat gpurun_out/fp64_peak.json
timeout 600 python bench.py --n 2048 --steps 1 --warmup 3 --cpu-sample-s 6 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_n1024.csv python bench.py --n 1024 --steps 1 --warmup 0 --no-cpu --no-accuracy --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log
