"""Summarise an ncu --page source --csv --print-source sass export: total
stall reasons and the hottest SASS instructions (with their stall mix).
usage: python tools/ncu_hot.py file.csv [top]"""
import csv
import sys
from collections import Counter

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0] != "Address"]
col = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for r in body:
    for s in stalls:
        try:
            tot[s] += float(r[col[s]] or 0)
        except ValueError:
            pass
allsamp = sum(tot.values())
print("total samples", allsamp)
for s, v in tot.most_common(12):
    print(f"  {s:28s} {v:10.0f} {100*v/max(allsamp,1):5.1f}%")
samp = col["Warp Stall Sampling (All Samples)"]
body.sort(key=lambda r: -float(r[samp] or 0))
print("\nhottest instructions:")
for r in body[:top]:
    v = float(r[samp] or 0)
    mix = sorted(((float(r[col[s]] or 0), s[6:]) for s in stalls), reverse=True)[:3]
    mixs = " ".join(f"{n}:{int(x)}" for x, n in mix if x > 0)
    print(f"{r[0]:>6s} {v:7.0f} {100*v/max(allsamp,1):5.1f}%  {r[1][:60]:60s} {mixs}")
