"""Per-sweep kernel time breakdown of a full block solve from an ncu launch
list (sweeps end at each k_block_norms launch).
usage: python tools/sweep_kernels.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and "Kernel Name" in r)
hdr = rows[hi]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
sweeps = [defaultdict(float)]
counts = [defaultdict(int)]
for r in rows[hi + 1:]:
    if len(r) != len(hdr) or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("hsvd::", "").replace("void ", "").split("<")[0]
    v = float(r[vi].replace(",", ""))
    unit = r[ui] if ui is not None else "ns"
    us = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
    sweeps[-1][name] += us
    counts[-1][name] += 1
    if name == "k_block_norms":
        sweeps.append(defaultdict(float))
        counts.append(defaultdict(int))
names = ["k_gram", "k_inner", "k_update"]
print("sweep | " + " | ".join(f"{k} ms (launches)" for k in names) + " | other ms")
for s, (d, c) in enumerate(zip(sweeps, counts)):
    if not d:
        continue
    other = sum(v for k, v in d.items() if k not in names)
    print(f"{s} | " + " | ".join(f"{d[k] / 1e3:.1f} ({c[k]})" for k in names) + f" | {other / 1e3:.2f}")
