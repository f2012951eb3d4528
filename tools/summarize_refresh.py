"""Summaries of a tools/gpu_refresh.sh run for profiles/: ncu tables of the
block kernels and the pointwise step kernel (from the raw CSV exports) and
the launch list.  usage: python tools/summarize_refresh.py TAG"""
import csv
import json
import os
import subprocess
import sys

tag = sys.argv[1]
out_dir = "profiles"
g = "gpurun_out"


def raw(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    recs = {}
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        name = r[h.index("Kernel Name")]
        recs.setdefault(name, r)
    return h, recs


METRICS = [
    ("grid", "launch__grid_size", None),
    ("block", "launch__block_size", None),
    ("gpu__time_duration (us)", "gpu__time_duration.sum", "{:.1f}"),
    ("dram__bytes_read (GB)", "dram__bytes_read.sum", "{:.3f}"),
    ("dram__bytes_write (GB)", "dram__bytes_write.sum", "{:.3f}"),
    ("DRAM throughput, % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "{:.1f}"),
    ("DMMA subpipe, % of peak sustained active",
     "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "{:.1f}"),
    ("FP64 pipe, % of peak sustained active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "{:.1f}"),
    ("registers / thread", "launch__registers_per_thread", None),
    ("IPC (SM, active)", "sm__inst_executed.avg.per_cycle_active", "{:.2f}"),
    ("shared-load bank conflicts (M)", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "m"),
    ("warps active, % of peak", "sm__warps_active.avg.pct_of_peak_sustained_active", "{:.1f}"),
]


def table(h, recs, order):
    cols = []
    for o in order:
        r = next((v for k, v in recs.items() if k.startswith("void " + o) or k.startswith(o)), None)
        cols.append((o, r))
    lines = ["| metric | " + " | ".join(o for o, _ in cols) + " |", "|---" * (len(cols) + 1) + "|"]
    for lab, key, fmt in METRICS:
        vals = []
        for _, r in cols:
            if r is None or key not in h:
                vals.append("n/a")
                continue
            v = r[h.index(key)]
            try:
                f = float(v)
                v = f"{f / 1e6:.2f}" if fmt == "m" else (fmt.format(f) if fmt else v)
            except ValueError:
                pass
            vals.append(v)
        lines.append(f"| {lab} | " + " | ".join(vals) + " |")
    return "\n".join(lines)


def bench(path):
    try:
        return json.loads(open(path).read().strip().splitlines()[-1])
    except Exception:  # noqa: BLE001
        return {}


bd, bp, br = bench(f"{g}/bench_default.json"), bench(f"{g}/bench_pointwise.json"), bench(f"{g}/bench_reference.json")
tests = open(f"{g}/pytest_gpu.log").read().strip().splitlines()[-1] if os.path.exists(f"{g}/pytest_gpu.log") else "?"
h, recs = raw(f"{g}/prof_block_raw.csv")
txt = [f"# {tag} -- ncu --set full of the block kernels, n=8192 p=4096, b=32", "",
       "Command (`tools/gpu_refresh.sh`, one GPU, one-stream step so every kernel covers all 128 slots):",
       "`ncu --set full --clock-control none --import-source on -k regex:\"k_update|k_gram|k_inner\" -s 40 -c 3 "
       "python tools/block_sweep.py 8192 1 32 full 1`. ncu times are cold-cache and serialised.", "",
       table(h, recs, ["k_gram_tma", "k_inner", "k_update"]), ""]
if bd:
    rf = bd.get("roofline", {})
    txt += [f"Bench line of the same box (`{tag}_bench_n8192.json`): block {bd['value']:.3f} s, e2e "
            f"{bd['e2e']['value']:.3f} s, {bd['sweeps']} sweeps, k_update at {100 * rf.get('frac', 0):.1f} % of the "
            f"sustained cuBLAS DGEMM measured in the same run, SM clock {bd['clocks']['sm_mhz']} MHz median "
            f"({', '.join(bd['clocks']['reasons']) or 'no throttle reason'})."]
if bp:
    txt += [f"Pointwise (bit-exact) line: {bp['value']:.2f} s, {100 * bp['roofline']['frac']:.1f} % of HBM "
            f"(`{tag}_bench_n8192_pointwise.json`)."]
if br:
    txt += [f"Reference arm: {br['value']:.0f} s (`{tag}_bench_reference.json`)."]
txt += [f"GPU test suite on the same box: {tests}"]
open(f"{out_dir}/{tag}_ncu_block_kernels.md", "w").write("\n".join(txt) + "\n")
if os.path.exists(f"{g}/prof_pointwise_raw.csv"):
    h2, recs2 = raw(f"{g}/prof_pointwise_raw.csv")
    open(f"{out_dir}/{tag}_ncu_pointwise.md", "w").write(
        f"# {tag} -- ncu --set full of the pointwise step kernel, n=8192 (sweep 0 step)\n\n"
        "`ncu --set full --clock-control none -k regex:\"k_pointwise_stream\" -s 20 -c 1 python tools/ncu_pointwise.py 8192`"
        " (cold-cache, serialised).\n\n" + table(h2, recs2, ["k_pointwise_stream"]) + "\n")
lt = subprocess.run([sys.executable, "tools/launch_table.py", f"{g}/launches_block.csv"], capture_output=True, text=True).stdout
open(f"{out_dir}/{tag}_launches_block.md", "w").write(
    f"# {tag} -- block mode, n=8192 p=4096: ncu launch list (first 1500 launches of one sweep, split streams)\n\n"
    "`tools/gpu_refresh.sh`; `python tools/launch_table.py gpurun_out/launches_block.csv`. Cold-cache, serialised: "
    "compare shares.\n\n" + lt)
for src, dst in [("bench_default.json", "bench_n8192.json"), ("bench_pointwise.json", "bench_n8192_pointwise.json"),
                 ("bench_reference.json", "bench_reference.json")]:
    if os.path.exists(f"{g}/{src}"):
        open(f"{out_dir}/{tag}_{dst}", "w").write(open(f"{g}/{src}").read())
print("\n".join(txt))
