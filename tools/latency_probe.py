"""Per-forward latency of the R50 presets across batch sizes (CUDA events on
the forward stream, graph replays after warm-up): the bs1 column is the
per-kernel fixed-cost floor (kernels per forward printed alongside)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_16733_b200 as ssn  # noqa: E402

batches = [int(b) for b in os.environ.get("BATCHES", "1,8,64").split(",")]
names = ["min", "mid", "max"]
desc = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, ssn.DTYPE_BF16, image_size=224, num_classes=1000,
                     max_batch=max(batches), input_format=ssn.INPUT_U8_NHWC)
eng = ssn.Engine(desc)
for i, n in enumerate(names):
    eng.register_subnet(i, ssn.ofa_resnet50_preset(n))
eng.prepare(batches)
x = torch.randint(0, 256, (max(batches), 224, 224, 3), dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for b in batches:
    row = []
    for i, n in enumerate(names):
        eng.actuate(i)
        for _ in range(5):
            eng.forward(x, b, b, None, stream=s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            eng.forward(x, b, b, None, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        row.append(f"{n} {e0.elapsed_time(e1) * 1000 / 20:8.1f} us ({eng.stats()['last_forward_kernels']} kernels)")
    print(f"bs{b:4d}: " + " | ".join(row), flush=True)
