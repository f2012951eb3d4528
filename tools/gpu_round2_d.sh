# round-2: TMA Gram -- probe, bit identity, bench A/B, block+sharded tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_gather_probe tools/tma_gather_probe.cu && timeout 60 ./tools/tma_gather_probe
timeout 900 python -m pytest tests/test_gpu_block.py -q -x -k "tma" 2>&1 | tail -3
timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_tma.json 2> gpurun_out/b_tma.err
HSVD_GRAM_TMA=0 timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_cpasync.json 2> gpurun_out/b_cpasync.err
python - <<'PY'
import json
for f in ("gpurun_out/b_tma.json", "gpurun_out/b_cpasync.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 4), d.get("sweeps"), d["roofline"].get("kernel_ms_sweep0"), [round(x, 1) for x in d.get("sweep_gpu_ms", [])])
    except Exception as e:
        print(f, "parse failed", e, open(f.replace('.json','.err')).read()[-800:])
PY
timeout 1200 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py -q 2>&1 | tail -3
