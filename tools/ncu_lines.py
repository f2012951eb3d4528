"""Per-source-line warp-stall samples from an ncu report exported with
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`.
usage: python tools/ncu_lines.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur, agg = None, {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 6 or not r[0].isdigit():
        continue
    # the source text may be split on commas: samples follow the two '-' columns
    k = next((i for i in range(1, len(r) - 2) if r[i] == "-" and r[i + 1] == "-"), None)
    if k is None:
        continue
    try:
        v = float(r[k + 2])
    except ValueError:
        continue
    agg[(cur, int(r[0]))] = (v, ",".join(r[1:k])[:110])
tot = sum(v for v, _ in agg.values())
print("total samples", tot)
for (f, ln), (v, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{ln:<5} {v:7.0f} {100 * v / tot:5.1f}%  {s}")
