"""First op whose output differs between two op-by-op runs of the same
input (debug aid for DESIGN.md §8's open issue)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_16733_b200 as ssn  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mid"
fam_name = sys.argv[2] if len(sys.argv) > 2 else "r50"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 64
fam = {"r50": ssn.FAMILY_OFA_RESNET50, "mbv3": ssn.FAMILY_OFA_MBV3, "bert": ssn.FAMILY_BERT}[fam_name]
size = 128 if fam == ssn.FAMILY_BERT else 224
desc = ssn.make_desc(fam, ssn.DTYPE_BF16, image_size=size,
                     num_classes=2 if fam == ssn.FAMILY_BERT else 1000, max_batch=B, seed=7,
                     input_format=ssn.INPUT_U8_NHWC)
eng = ssn.Engine(desc)
cfg = ssn.supernets.preset(fam, name)
eng.register_subnet(0, cfg)
eng.prepare([B])
eng.actuate(0)
rng = np.random.default_rng(7)
if fam == ssn.FAMILY_BERT:
    x = rng.integers(0, 30522, size=(B, size), dtype=np.int32)
else:
    x = rng.integers(0, 256, size=(B, size, size, 3), dtype=np.uint8)
eng.infer(x, B, B)
runs = [eng.debug_op_checksums(0, B) for _ in range(3)]
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
