mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -4
for i in 1 2; do
timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_tile$i.json 2> gpurun_out/b_tile$i.err
done
python - <<'PY'
import json
for f in ("gpurun_out/b_tile1.json", "gpurun_out/b_tile2.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 4), d.get("sweeps"), d["roofline"].get("kernel_ms_sweep0"), [round(x, 1) for x in d.get("sweep_gpu_ms", [])], round(d["e2e"]["value"], 4))
    except Exception as e:
        print(f, "parse failed", e, open(f.replace('.json','.err')).read()[-1500:])
PY
