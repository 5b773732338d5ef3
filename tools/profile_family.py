"""Per-subnet latency / throughput table for one supernet family on cuda:0
(min/mid/max presets, CUDA-graph replay timed by ssn_profile_latency).

    python tools/profile_family.py --family bert --batches 1,8,32,64
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_16733_b200 as ssn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="bert", choices=["r50", "mbv3", "bert"])
ap.add_argument("--batches", default="1,8,32,64")
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--out", default="")
a = ap.parse_args()
fam = {"r50": ssn.FAMILY_OFA_RESNET50, "mbv3": ssn.FAMILY_OFA_MBV3, "bert": ssn.FAMILY_BERT}[a.family]
size = 128 if fam == ssn.FAMILY_BERT else 224
batches = [int(b) for b in a.batches.split(",")]
desc = ssn.make_desc(fam, ssn.DTYPE_BF16, image_size=size,
                     num_classes=2 if fam == ssn.FAMILY_BERT else 1000, max_batch=max(batches))
eng = ssn.Engine(desc)
names = ["min", "mid", "max"]
for i, n in enumerate(names):
    eng.register_subnet(i, ssn.supernets.preset(fam, n))
eng.prepare(batches)
rows = []
for i, n in enumerate(names):
    cost = ssn.plan_cost(desc, ssn.supernets.preset(fam, n))
    for b in batches:
        us = eng.profile_latency(i, b, a.iters)
        tf = cost["flops"] * b / (us * 1e-6) / 1e12
        rows.append({"family": a.family, "subnet": n, "batch": b, "us": round(us, 1),
                     "items_per_s": round(b / (us * 1e-6), 1),
                     "gflop_per_item": round(cost["flops"] / 1e9, 3), "tflops": round(tf, 1)})
        print(json.dumps(rows[-1]))
if a.out:
    with open(a.out, "w") as f:
        json.dump(rows, f, indent=1)
