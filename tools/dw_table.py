"""Summarise an ncu --metrics CSV of depthwise launches: time, DRAM bytes, GB/s."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
k = collections.OrderedDict()
for r in rows[1:]:
    k.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]][:30]})[r[ix["Metric Name"]]] = r[ix["Metric Value"]]
tt = 0.0
for v in k.values():
    g = lambda m: float(v.get(m, "0").replace(",", ""))
    t = g("gpu__time_duration.sum")
    tt += t
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    print(f"{v['name'][:22]} grid={v.get('launch__grid_size', '?'):>7} t={t / 1e3:7.1f}us "
          f"rd={rd / 1e6:7.1f}MB wr={wr / 1e6:7.1f}MB GB/s={(rd + wr) / t:6.0f} "
          f"sm%={v.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', '?')} "
          f"fma%={v.get('sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', '?')}")
print(f"total {tt / 1e3:.1f} us")
