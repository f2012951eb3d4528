mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
HSVD_PLAN_STATS=1 python tools/block_telemetry.py 8192 2>&1 | tail -3
for ls in 1 0; do
HSVD_LATE_SPLIT=$ls timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_ls$ls.json 2> gpurun_out/b_ls$ls.err
done
python - <<'PY'
import json
for f in ("gpurun_out/b_ls1.json", "gpurun_out/b_ls0.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 4), d.get("sweeps"), d["gpu_launches"], [round(x, 1) for x in d.get("sweep_gpu_ms", [])])
    except Exception as e:
        print(f, "parse failed", e, open(f.replace('.json','.err')).read()[-1500:])
PY
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -2
