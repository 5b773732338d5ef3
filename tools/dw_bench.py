"""Depthwise operator microbenchmark (ssn_op_dw_bf16) on cuda:0.

    python tools/dw_bench.py 256,56,56,96,192,7,3,1      # n,h,w,c,c_max,k_max,k,stride
Prints device time per launch (CUDA events over --iters launches) and the
achieved algorithmic HBM GB/s (input + output bytes, bf16)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_16733_b200 as ssn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("shapes", nargs="+")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--act", type=int, default=1)
a = ap.parse_args()
dev = torch.device("cuda:0")
for sh in a.shapes:
    n, h, w, c, c_max, k_max, k, s = (int(v) for v in sh.split(","))
    pad = k // 2
    ho, wo = (h + 2 * pad - k) // s + 1, (w + 2 * pad - k) // s + 1
    x = torch.randn(n, h, w, c, device=dev).to(torch.bfloat16)
    wt = (torch.randn(k_max, k_max, c_max, device=dev) / k).to(torch.bfloat16)
    sc = torch.rand(c, device=dev) + 0.5
    sf = torch.rand(c, device=dev) - 0.5
    y = torch.empty(n, ho, wo, c, device=dev, dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        ssn.op_dw_bf16(x, n, h, w, c, wt, c_max, k_max, k, s, sc, sf, a.act, y, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.iters):
        ssn.op_dw_bf16(x, n, h, w, c, wt, c_max, k_max, k, s, sc, sf, a.act, y, st)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.iters
    byts = 2 * (n * h * w * c + n * ho * wo * c)
    fma = n * ho * wo * c * k * k
    print(f"dw {sh}: {us:8.1f} us  {byts / us / 1e3:7.0f} GB/s  {fma / us / 1e6:6.2f} TFMA/s")
