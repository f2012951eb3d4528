mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { tag=$1; shift; env "$@" timeout 400 python bench.py --steps 2 --warmup 3 --no-cpu --no-accuracy $BARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{tag}.json").read().strip().splitlines()[-1])
    print(f"{tag:12s} {d['value']:.4f} sweeps {d['sweeps']} {[round(x, 1) for x in d.get('sweep_gpu_ms', [])]}")
except Exception as e:
    print(tag, "failed", e)
PY
}
run reuse1a HSVD_REUSE=1
run reuse0a HSVD_REUSE=0
run reuse1b HSVD_REUSE=1
run reuse0b HSVD_REUSE=0
BARGS="--inner-ordering oriented" run oriented HSVD_REUSE=1
BARGS="--block-cols 16" run b16 HSVD_REUSE=1
