# pointwise bit-exactness after the V-batch change + a pointwise bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_xl.py -q -k "not block" --timeout=900 --timeout-method=thread 2>&1 | tail -3
timeout 900 python bench.py --mode pointwise --steps 1 --warmup 1 --no-cpu --no-accuracy > gpurun_out/b_pw.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_pw.json').read().strip().splitlines()[-1]); print(d['value'], d['sweeps'], d['roofline'].get('frac'), d['roofline'].get('achieved'))"
