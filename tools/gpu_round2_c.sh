# round-2: bench with/without all-skip reuse, then the full GPU suite
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_reuse.json 2> gpurun_out/b_reuse.err
HSVD_REUSE=0 timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_noreuse.json 2> gpurun_out/b_noreuse.err
python - <<'PY'
import json
for f in ("gpurun_out/b_reuse.json", "gpurun_out/b_noreuse.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 4), d.get("sweeps"), d["roofline"].get("kernel_ms_sweep0"), [round(x, 1) for x in d.get("sweep_gpu_ms", [])])
    except Exception as e:
        print(f, "parse failed", e)
PY
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
