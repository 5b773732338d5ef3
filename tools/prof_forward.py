"""Minimal driver for ncu captures: the bench's sweep step (actuate + forward
of min/mid/max at one batch), W untimed warm-up steps then S steps."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_16733_b200 as ssn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--image", type=int, default=224)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--subnets", default="min,mid,max")
ap.add_argument("--family", default="r50", choices=["r50", "mbv3", "bert"])
a = ap.parse_args()
names = a.subnets.split(",")
fam = {"r50": ssn.FAMILY_OFA_RESNET50, "mbv3": ssn.FAMILY_OFA_MBV3, "bert": ssn.FAMILY_BERT}[a.family]
if fam == ssn.FAMILY_BERT:
    a.image = 128  # sequence length
desc = ssn.make_desc(fam, ssn.DTYPE_BF16, image_size=a.image,
                     num_classes=2 if fam == ssn.FAMILY_BERT else 1000, max_batch=a.batch,
                     input_format=ssn.INPUT_U8_NHWC)
eng = ssn.Engine(desc)
for i, n in enumerate(names):
    eng.register_subnet(i, ssn.supernets.preset(fam, n))
eng.prepare([a.batch])
if fam == ssn.FAMILY_BERT:
    x = torch.randint(0, 30522, (a.batch, a.image), dtype=torch.int32, device="cuda")
else:
    x = torch.randint(0, 256, (a.batch, a.image, a.image, 3), dtype=torch.uint8, device="cuda")
for it in range(a.warmup + a.steps):
    for i in range(len(names)):
        eng.actuate(i)
        eng.forward(x, a.batch, a.batch, None)
    eng.synchronize()
print("kernels per forward:", eng.stats()["last_forward_kernels"])
