"""Forward the same bs64 batch twice and report rows that differ (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_16733_b200 as ssn  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "max"
desc = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, ssn.DTYPE_BF16, image_size=224, num_classes=1000,
                     max_batch=64, seed=7, input_format=ssn.INPUT_U8_NHWC)
eng = ssn.Engine(desc)
eng.register_subnet(0, ssn.ofa_resnet50_preset(name))
eng.prepare([64])
eng.actuate(0)
x = np.random.default_rng(7).integers(0, 256, size=(64, 224, 224, 3), dtype=np.uint8)
a = eng.infer(x, 64, 64)
for it in range(3):
    b = eng.infer(x, 64, 64)
    diff = ~((a == b) | (np.isnan(a) & np.isnan(b)))
    rows = np.where(diff.any(1))[0]
    print(name, "run", it, "rows differing:", rows.tolist()[:20],
          "finite rows among them:", [int(r) for r in rows if np.isfinite(a[r]).all() and np.isfinite(b[r]).all()][:10],
          "max |a|:", float(np.nanmax(np.abs(a[rows]))) if len(rows) else 0.0)
