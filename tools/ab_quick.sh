# quick A/B: build, one n=8192 bench line, the block + sharded GPU tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-accuracy ${BENCH_ARGS} > /tmp/b.json 2> /tmp/b.err || tail -5 /tmp/b.err
python - <<'PY'
import json
try:
    d = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
    print(round(d['value'], 4), d.get('sweeps'), d['roofline'].get('kernel_ms_sweep0'), [round(x, 1) for x in d.get('sweep_gpu_ms', [])])
except Exception as e:
    print('bench parse failed', e)
PY
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -3
