"""Per-opcode executed-instruction / stall histogram of an ncu report's SASS
source page:  python tools/ncu_sass_hist.py report.ncu-rep [top_lines]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc = h.index("Address"), h.index("Source")
ie, iss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = 0
byop, stall = collections.Counter(), collections.Counter()
data = []
for r in rows[2:]:
    try:
        n, s = int(r[ie]), int(r[iss])
    except (ValueError, IndexError):
        continue
    toks = r[isrc].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    byop[op] += n
    stall[op] += s
    tot += n
    data.append((n, s, r[ia][-5:], r[isrc].strip()))
print("instructions executed", tot)
for op, n in byop.most_common(22):
    print(f"{op:10s} {n:12d} {n / tot * 100:5.1f}%  stall samples {stall[op]}")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
data.sort(key=lambda x: -x[1])
for d in data[:top]:
    print(d)
