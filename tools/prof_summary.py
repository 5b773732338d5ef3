"""Aggregate '[conv_tc prof]' lines (SSN_TC_DEBUG & 32) from stdin: mean
total / wait / wait2 cycles per (tiles, nk, warp)."""
import collections
import re
import sys

acc = collections.defaultdict(lambda: [0, 0, 0, 0])
for line in sys.stdin:
    m = re.search(r"tiles=(\d+) nk=(\d+) warp=(\d+) total=(\d+) wait=(\d+) wait2=(\d+)", line)
    if not m:
        continue
    k = (int(m[1]), int(m[2]), int(m[3]))
    a = acc[k]
    a[0] += 1
    a[1] += int(m[4])
    a[2] += int(m[5])
    a[3] += int(m[6])
for k, a in sorted(acc.items()):
    n = a[0]
    print(f"tiles={k[0]} nk={k[1]} warp={k[2]} n={n} total={a[1] / n:.0f} wait={a[2] / n:.0f} "
          f"wait2={a[3] / n:.0f} busy={(a[1] - a[2] - a[3]) / n:.0f}")
