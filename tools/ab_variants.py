"""A/B compile-time variants on the GPU box: for each -D set, rebuild the
library in-tree, run one short bench line, print value, kernel split of the
profiled sweep 0 and the per-sweep times.  Restores the default build.

    python tools/ab_variants.py "A:" "B:-DHSVD_GRAM_NSEG=8" ...
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_1008_1371_b200 import _build  # noqa: E402

BASE = list(_build.COMMON)
args = sys.argv[1:]
extra_bench = os.environ.get("BENCH_ARGS", "").split()
script = os.environ.get("AB_SCRIPT")  # run this script instead of bench.py (prints its last line)
for spec in args + ["default:"]:
    name, _, flags = spec.partition(":")
    _build.COMMON[:] = BASE + flags.split()
    _build.build(force=True)
    if name == "default":
        break
    if script:
        out = subprocess.run([sys.executable, *script.split()], capture_output=True, text=True,
                             timeout=600)
        print(f"{name:10s} {flags:40s} {out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]}",
              flush=True)
        continue
    out = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "1", "--no-cpu",
                          "--no-accuracy", *extra_bench], capture_output=True, text=True, timeout=600)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        print(f"{name:10s} {flags:40s} value {d['value']:.4f} sweeps {d['sweeps']} "
              f"k0 {d['roofline'].get('kernel_ms_sweep0')} "
              f"sw {[round(x, 1) for x in d.get('sweep_gpu_ms', [])]}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(name, "failed", e, out.stderr[-1500:], flush=True)
