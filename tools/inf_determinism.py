"""Op-level bit-reproducibility with non-finite inputs (debug aid for the
open issue in DESIGN.md §8): each conv path runs twice on an activation
sprinkled with +-inf; outputs must match bit for bit (NaN positions too)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_16733_b200 as ssn  # noqa: E402

CASES = [  # n, h, w, cin, cin_max, cout, cout_max, k, stride, residual
    (8, 56, 56, 88, 88, 88, 88, 3, 1, 0),      # halo
    (8, 112, 112, 32, 32, 32, 32, 3, 1, 1),    # halo + residual
    (8, 56, 56, 88, 88, 256, 256, 1, 1, 1),    # resident B
    (8, 14, 14, 360, 360, 360, 360, 3, 1, 0),  # im2col, pairs
    (8, 28, 28, 176, 176, 512, 512, 1, 1, 1),  # streamed B
    (8, 7, 7, 720, 720, 720, 720, 3, 2, 0),    # stride 2
]
torch.manual_seed(0)
for c in CASES:
    n, h, w, cin, cin_max, cout, cout_max, k, st, has_res = c
    pad = k // 2
    ho, wo = (h + 2 * pad - k) // st + 1, (w + 2 * pad - k) // st + 1
    x = torch.randn(n, h, w, cin, device="cuda")
    mask = torch.rand_like(x) < 0.01
    x[mask] = float("inf")
    x[torch.rand_like(x) < 0.005] = float("-inf")
    x = x.to(torch.bfloat16)
    wt = (torch.randn(cout_max, k, k, cin_max, device="cuda") * 0.05).to(torch.bfloat16)
    sc = torch.ones(cout, device="cuda")
    sh = torch.zeros(cout, device="cuda")
    res = torch.randn(n, ho, wo, cout, device="cuda").to(torch.bfloat16) if has_res else None
    outs = []
    for _ in range(3):
        y = torch.full((n, ho, wo, cout), 7.0, device="cuda", dtype=torch.bfloat16)
        ssn.op_conv_bf16(x, n, h, w, cin, wt, cout_max, cin_max, k, st, pad, cout, sc, sh, res, 1, 0, y)
        torch.cuda.synchronize()
        outs.append(y.view(torch.int16).clone())
    same = all(torch.equal(outs[0], o) for o in outs[1:])
    ndiff = max(int((outs[0] != o).sum()) for o in outs[1:])
    print(c, "bit-identical" if same else f"DIFFERS ({ndiff} elements)", flush=True)
