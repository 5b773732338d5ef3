"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
for d in data:
    name = d["Kernel Name"].split("(")[0][:48]
    v = float(d["Metric Value"].replace(",", "")) / 1e3
    agg[name][0] += 1
    agg[name][1] += v
    seq.append((name, v, d.get("Grid Size", "")))
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:10.1f} us {100 * v[1] / tot:5.1f}% n={v[0]:4d} {k}")
print(f"total {tot:.1f} us over {len(data)} launches")
for s in seq[-last:] if last else []:
    print(f"{s[1]:8.1f} {s[2]:>14} {s[0]}")
