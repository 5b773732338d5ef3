"""Per-launch table from an `ncu --metrics ... --csv` launch list (one row per
metric): kernel, grid, device time, DRAM read/write bytes (the bench
roofline's `traffic`), tensor-pipe / DRAM / L2 throughput %.  The summary line
gives the conv_tc mean DRAM bytes per launch.

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,\
gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,\
lts__t_sectors.avg.pct_of_peak_sustained_elapsed,launch__grid_size --csv ...
"""
import collections
import csv
import json
import sys

SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
launches = collections.OrderedDict()
for r in rows[1:]:
    d = launches.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]].split("(")[0]
                                          .replace("void ", "").replace("ssn::", "")})
    v = r[ix["Metric Value"]].replace(",", "")
    u = r[ix["Metric Unit"]] if "Metric Unit" in ix else ""
    try:
        d[r[ix["Metric Name"]]] = float(v) * SCALE.get(u, 1.0)
    except ValueError:
        d[r[ix["Metric Name"]]] = v
cols = [("us", "gpu__time_duration.sum"), ("dram_rd_MB", "dram__bytes_read.sum"),
        ("dram_wr_MB", "dram__bytes_write.sum"),
        ("tensor%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("l2%", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed")]
print("| # | kernel | grid | " + " | ".join(c for c, _ in cols) + " |")
print("|---|---|---|" + "---|" * len(cols))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for n, d in enumerate(launches.values()):
    print(f"| {n} | {d['name']} | {d.get('launch__grid_size', '?')} | " +
          " | ".join(f"{d.get(m, float('nan')):.1f}" if isinstance(d.get(m), float) else "?"
                     for _, m in cols) + " |")
    fam = d["name"].split("<")[0]
    a = agg[fam]
    a[0] += 1
    a[1] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    a[2] += d.get("gpu__time_duration.sum", 0.0)
summary = {k: {"launches": v[0], "dram_MB_per_launch": round(v[1] / v[0], 3),
               "us_per_launch": round(v[2] / v[0], 2)} for k, v in agg.items()}
print("\n" + json.dumps(summary))
