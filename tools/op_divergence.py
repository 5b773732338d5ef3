"""First op whose output differs between two op-by-op runs of the same
input (debug aid for DESIGN.md §8's open issue)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_16733_b200 as ssn  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mid"
desc = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, ssn.DTYPE_BF16, image_size=224, num_classes=1000,
                     max_batch=64, seed=7, input_format=ssn.INPUT_U8_NHWC)
eng = ssn.Engine(desc)
cfg = ssn.ofa_resnet50_preset(name)
eng.register_subnet(0, cfg)
eng.prepare([64])
eng.actuate(0)
x = np.random.default_rng(7).integers(0, 256, size=(64, 224, 224, 3), dtype=np.uint8)
eng.infer(x, 64, 64)
runs = [eng.debug_op_checksums(0, 64) for _ in range(3)]
rows = ssn.supernets.plan_ops(desc, cfg)
for i in range(len(rows)):
    vals = {int(r[i]) for r in runs}
    if len(vals) > 1:
        r = rows[i]
        print("first diverging op", i, r["kind"], "k", r["k"], "s", r["stride"], r["cin"], "->", r["cout"],
              "hw", r["hout"], "res", r["has_residual"])
        break
else:
    print("op-by-op runs identical;", sum(1 for v in runs[0] if v), "ops hashed")
