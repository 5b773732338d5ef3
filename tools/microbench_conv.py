"""Time single WeightSlice convs through ssn_op_conv_bf16 (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_16733_b200 as ssn  # noqa: E402

CASES = [  # n, h, w, cin, cin_max, cout, cout_max, k, stride
    (64, 112, 112, 24, 32, 40, 64, 3, 1),
    (64, 224, 224, 8, 8, 24, 32, 3, 2),
    (64, 56, 56, 88, 88, 88, 88, 3, 1),
    (64, 14, 14, 360, 360, 360, 360, 3, 1),
    (64, 56, 56, 88, 88, 256, 256, 1, 1),
    (64, 28, 28, 512, 512, 176, 176, 1, 1),
]
only = os.environ.get("CASES")
for ci, c in enumerate(CASES):
    if only and str(ci) not in only.split(","):
        continue
    n, h, w, cin, cin_max, cout, cout_max, k, st = c
    pad = k // 2
    ho, wo = (h + 2 * pad - k) // st + 1, (w + 2 * pad - k) // st + 1
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    wt = (torch.randn(cout_max, k, k, cin_max, device="cuda") * 0.05).to(torch.bfloat16)
    sc = torch.ones(cout, device="cuda")
    sh = torch.zeros(cout, device="cuda")
    y = torch.empty(n, ho, wo, cout, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        ssn.op_conv_bf16(x, n, h, w, cin, wt, cout_max, cin_max, k, st, pad, cout, sc, sh, None, 1, 0, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 10
    e0.record()
    for _ in range(it):
        ssn.op_conv_bf16(x, n, h, w, cin, wt, cout_max, cin_max, k, st, pad, cout, sc, sh, None, 1, 0, y)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / it
    flops = 2 * n * ho * wo * cout * cin * k * k
    byts = 2 * (n * h * w * cin + n * ho * wo * cout)
    print(f"dbg={os.environ.get('SSN_TC_DEBUG', '0')} case{ci} {c}: {us:8.1f} us  "
          f"{flops / us / 1e6:7.1f} TF/s  {byts / us / 1e3:7.1f} GB/s", flush=True)
