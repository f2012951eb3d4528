"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list into a
markdown table of per-kernel launches, total time and share.
usage: python tools/launch_table.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and "Kernel Name" in r)
hdr = rows[hi]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hi + 1:]:
    if len(r) != len(hdr) or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("hsvd::", "")
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
    us = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
    tot[name] += us
    cnt[name] += 1
all_us = sum(tot.values())
print("| kernel | launches | total us | share | avg us |")
print("|---|---|---|---|---|")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {100 * tot[k] / all_us:.1f}% | {tot[k] / cnt[k]:.2f} |")
