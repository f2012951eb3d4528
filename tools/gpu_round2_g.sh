mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_block.py -q -x -k "tma or reuse or deterministic or matches_reference" 2>&1 | tail -3
timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_g.json 2> gpurun_out/b_g.err
HSVD_REUSE=0 timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy > gpurun_out/b_g0.json 2> gpurun_out/b_g0.err
python - <<'PY'
import json
for f in ("gpurun_out/b_g.json", "gpurun_out/b_g0.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 4), d.get("sweeps"), d["roofline"].get("kernel_ms_sweep0"), [round(x, 1) for x in d.get("sweep_gpu_ms", [])], d["roofline"].get("peak"), d["roofline"].get("peak_burst"), d["roofline"].get("frac"))
    except Exception as e:
        print(f, "parse failed", e, open(f.replace('.json','.err')).read()[-1500:])
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_tma" \
    -s 20 -c 1 -o gpurun_out/prof_gram_tma2 python tools/block_sweep.py 8192 1 32 full 1 > gpurun_out/ncu_gram.log 2>&1
ncu -i gpurun_out/prof_gram_tma2.ncu-rep --page raw --csv > gpurun_out/prof_gram_tma2_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_gram_tma2.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_gram_tma2_src.csv 2>/dev/null
python tools/ncu_hot.py gpurun_out/prof_gram_tma2_src.csv 12 > gpurun_out/prof_gram_tma2_hot.txt 2>&1
head -30 gpurun_out/prof_gram_tma2_hot.txt
