"""Time single WeightSlice convs through ssn_op_conv_bf16 (CUDA events).

SSN_TC_DEBUG=1 drops the epilogue's global traffic, =2 drops the MMAs, =3
both: the difference isolates which stage bounds a layer (profiling only).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_16733_b200 as ssn  # noqa: E402

CASES = [  # n, h, w, cin, cin_max, cout, cout_max, k, stride, residual
    (64, 112, 112, 24, 32, 40, 64, 3, 1, 0),
    (64, 56, 56, 88, 88, 88, 88, 3, 1, 0),
    (64, 14, 14, 360, 360, 360, 360, 3, 1, 0),
    (64, 56, 56, 88, 88, 256, 256, 1, 1, 1),
    (64, 56, 56, 256, 256, 88, 88, 1, 1, 0),
    (64, 14, 14, 360, 360, 1024, 1024, 1, 1, 1),
    (64, 7, 7, 720, 720, 720, 720, 3, 1, 0),
    (64, 7, 7, 2048, 2048, 720, 720, 1, 1, 0),
    (64, 28, 28, 176, 176, 176, 176, 3, 1, 0),
    (1, 7, 7, 64, 64, 64, 64, 1, 1, 0),
    (8, 14, 14, 64, 64, 64, 64, 1, 1, 0),
    (64, 56, 56, 56, 88, 56, 88, 3, 1, 0),
    (1, 14, 14, 16, 16, 16, 16, 3, 1, 0),
    (1, 56, 56, 88, 88, 88, 88, 3, 1, 0),
    (64, 56, 56, 88, 88, 256, 256, 1, 1, 0),   # case3 without the residual
    (64, 56, 56, 256, 256, 256, 256, 1, 1, 0), # wide in, wide out
    (256, 14, 14, 2048, 2048, 2048, 2048, 1, 1, 0),  # compute-bound GEMM probe
    (256, 14, 14, 512, 512, 512, 512, 3, 1, 0),      # compute-bound 3x3 probe
    (64, 7, 7, 2048, 2048, 720, 720, 1, 1, 0),       # = case7 (small M)
    (64, 14, 14, 136, 360, 136, 360, 3, 1, 0),       # min-subnet 14px 3x3
    (64, 14, 14, 136, 384, 136, 384, 3, 1, 0),       # 20: aligned weights, misaligned act
    (64, 14, 14, 192, 384, 192, 384, 3, 1, 0),       # 21: aligned both
    (64, 14, 14, 192, 360, 192, 360, 3, 1, 0),       # 22: aligned act, misaligned weights
    (64, 14, 14, 384, 384, 384, 384, 3, 1, 0),       # 23: case2 but aligned
    (64, 7, 7, 2048, 2048, 768, 768, 1, 1, 0),       # 24: case7, N aligned to 256
    (256, 14, 14, 512, 512, 384, 384, 3, 1, 0),      # 25: bn128 pair tiles, long grid
    (256, 14, 14, 360, 360, 360, 360, 3, 1, 0),      # 26: case2 at n=256
    (16, 14, 14, 360, 360, 360, 360, 3, 1, 0),       # 27: case2 at n=16
    (256, 14, 14, 2048, 2048, 384, 384, 1, 1, 0),    # 28: bn128 pairs, tiled A (vs 25: im2col A)
    (256, 14, 14, 4608, 4608, 384, 384, 1, 1, 0),    # 29: = case25 as a 1x1 (same M, N, K)
    (64, 14, 14, 360, 360, 1024, 1024, 1, 1, 0),     # 30: stage-3 expand, no residual
    (64, 7, 7, 720, 720, 2048, 2048, 1, 1, 0),       # 31: stage-4 expand
    (64, 14, 14, 1024, 1024, 360, 360, 1, 1, 0),     # 32: stage-3 reduce
    (64, 112, 112, 32, 32, 64, 64, 3, 1, 0),         # 33: max stem 3x3 32->64 (halo)
    (64, 112, 112, 32, 32, 32, 32, 3, 1, 1),         # 34: stem residual block (halo + residual)
    (64, 14, 14, 368, 368, 368, 368, 3, 1, 0),       # 35: case2 at a 32-B aligned width
    (64, 7, 7, 768, 768, 768, 768, 3, 1, 0),         # 36: case6 at a 128-B aligned width
    (64, 28, 28, 192, 192, 192, 192, 3, 1, 0),       # 37: case8 at a 128-B aligned width
    (64, 14, 14, 352, 352, 352, 352, 3, 1, 0),       # 38: 32-B aligned, narrower than case2
    (64, 14, 14, 1024, 1024, 368, 368, 1, 1, 0),     # 39: = case32 at a 32-B aligned width
    (64, 14, 14, 1024, 1024, 384, 384, 1, 1, 0),     # 40: = case32 at a 128-B aligned width
    (64, 14, 14, 384, 384, 1024, 1024, 1, 1, 1),     # 41: = case5 with an aligned input
    (64, 14, 14, 360, 368, 360, 360, 3, 1, 0),       # 42: case2 with 32-B weight rows (engine store)
    (64, 14, 14, 1024, 1024, 360, 360, 1, 1, 0),     # 43: = case32 (aligned weights already)
    (64, 14, 14, 360, 368, 1024, 1024, 1, 1, 1),     # 44: case5 with 32-B weight rows
    (256, 14, 14, 360, 368, 360, 360, 3, 1, 0),      # 45: case26 with 32-B weight rows
    (64, 28, 28, 360, 360, 360, 360, 3, 2, 0),       # 46: max stage-3 stride-2 3x3 (28 -> 14 px)
    (64, 56, 56, 176, 176, 176, 176, 3, 2, 0),       # 47: max stage-2 stride-2 3x3 (56 -> 28 px)
    (64, 14, 14, 720, 720, 720, 720, 3, 2, 0),       # 48: max stage-4 stride-2 3x3 (14 -> 7 px)
    (64, 56, 56, 64, 64, 256, 256, 1, 1, 0),         # 49: max stage-1 downsample / expand-sized 1x1 (HBM-bound)
]
only = os.environ.get("CASES")
for ci, c in enumerate(CASES):
    if only and str(ci) not in only.split(","):
        continue
    n, h, w, cin, cin_max, cout, cout_max, k, st, has_res = c
    pad = k // 2
    ho, wo = (h + 2 * pad - k) // st + 1, (w + 2 * pad - k) // st + 1
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    wt = (torch.randn(cout_max, k, k, cin_max, device="cuda") * 0.05).to(torch.bfloat16)
    sc = torch.ones(cout, device="cuda")
    sh = torch.zeros(cout, device="cuda")
    y = torch.empty(n, ho, wo, cout, device="cuda", dtype=torch.bfloat16)
    res = torch.randn(n, ho, wo, cout, device="cuda").to(torch.bfloat16) if has_res else None
    for _ in range(3):
        ssn.op_conv_bf16(x, n, h, w, cin, wt, cout_max, cin_max, k, st, pad, cout, sc, sh, res, 1, 0, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 10
    e0.record()
    for _ in range(it):
        ssn.op_conv_bf16(x, n, h, w, cin, wt, cout_max, cin_max, k, st, pad, cout, sc, sh, res, 1, 0, y)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / it
    flops = 2 * n * ho * wo * cout * cin * k * k
    byts = 2 * (n * h * w * cin + n * ho * wo * cout * (2 if has_res else 1))
    roof = max(flops / 1.4e6, byts / 6.5e3)
    print(f"dbg={os.environ.get('SSN_TC_DEBUG', '0')} case{ci} {c}: {us:8.1f} us  "
          f"{flops / us / 1e6:7.1f} TF/s  {byts / us / 1e3:7.1f} GB/s  roof {roof:6.1f} us "
          f"frac {roof / us:.2f}", flush=True)
