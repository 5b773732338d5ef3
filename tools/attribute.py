"""Attribute an ncu launch list (tools/prof_forward.py run) to plan ops.

Each forward launches set_row (on a switch), then the plan's active ops in
order.  For every op: measured µs, algorithmic GFLOP / MB, the roofline time
max(flops / tc_peak, bytes / hbm_peak) and the fraction achieved.

usage: python tools/attribute.py launches.csv --subnets min,mid,max --batch 64
"""
import argparse
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_16733_b200 as ssn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--subnets", default="min,mid,max")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--image", type=int, default=224)
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--family", default="r50", choices=["r50", "mbv3"])
ap.add_argument("--json", default="")
a = ap.parse_args()

peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
TC, HBM = peaks["bf16_tflops"] * 1e12, peaks["hbm_gbs"] * 1e9

rows = list(csv.reader(open(a.csv)))
hdr, launches = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        if "ssn::" not in name:
            continue
        launches.append((name, float(d["Metric Value"].replace(",", "")) / 1e3))

fam = ssn.FAMILY_OFA_MBV3 if a.family == "mbv3" else ssn.FAMILY_OFA_RESNET50
desc = ssn.make_desc(fam, image_size=a.image, max_batch=a.batch)
names = a.subnets.split(",")
per_fwd = []
for n in names:
    cost = ssn.plan_cost(desc, ssn.supernets.preset(fam, n))
    ops = [p for p in cost["per_op"] if p is not None]
    # bf16 stem: the input op launches nothing (fused into the stem conv)
    if os.environ.get("SSN_TC_DEBUG", "0") == "0" and ops and ops[0]["op"] == "input" \
            and len(ops) > 1 and ops[1]["cin"] == 3:
        ops = ops[1:]
    per_fwd.append((n, ops))
# the last len(names) forwards in the list are the measured step
need = sum(len(ops) for _, ops in per_fwd)
ops_launches = []
for l in launches:
    if "set_row" in l[0]:
        continue
    if "conv_finish_kernel" in l[0] and ops_launches:  # split-K tail of the previous conv
        ops_launches[-1] = (ops_launches[-1][0], ops_launches[-1][1] + l[1])
        continue
    ops_launches.append(l)
ops_launches = ops_launches[-need:]
out, k = [], 0
for n, ops in per_fwd:
    for p in ops:
        kname, us = ops_launches[k]
        k += 1
        f = p["flops"] * a.batch
        b = p["bytes"] * a.batch + p["weight_bytes"]
        roof = max(f / TC, b / HBM) * 1e6
        out.append(dict(subnet=n, op=p["op"], k=p["k"], stride=p["stride"], cin=p["cin"],
                        cout=p["cout"], hw=p["hout"], us=us, gflop=f / 1e9, mb=b / 1e6,
                        roof_us=roof, frac=roof / us if us else 0, kernel=kname.split("::")[-1]))
tot = sum(o["us"] for o in out)
troof = sum(o["roof_us"] for o in out)
print(f"total {tot:.1f} us, roofline {troof:.1f} us, frac {troof / tot:.3f}")
for n in names:
    s = [o for o in out if o["subnet"] == n]
    print(f"  {n}: {sum(o['us'] for o in s):8.1f} us  roof {sum(o['roof_us'] for o in s):7.1f}")
print(f"{'subnet':6} {'op':7} {'k':>2} {'s':>2} {'cin':>5} {'cout':>5} {'hw':>4} {'us':>8} "
      f"{'roof':>7} {'frac':>5} {'GF':>6} {'MB':>7} {'lost':>7}")
for o in sorted(out, key=lambda o: -(o["us"] - o["roof_us"]))[:a.top]:
    print(f"{o['subnet']:6} {o['op']:7} {o['k']:2d} {o['stride']:2d} {o['cin']:5d} {o['cout']:5d} "
          f"{o['hw']:4d} {o['us']:8.1f} {o['roof_us']:7.1f} {o['frac']:5.2f} {o['gflop']:6.1f} "
          f"{o['mb']:7.1f} {o['us'] - o['roof_us']:7.1f}")
if a.json:
    json.dump(out, open(a.json, "w"), indent=1)
