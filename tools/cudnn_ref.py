"""Library yardstick (profiling only, never the product path): time cuDNN
(torch.nn.functional.conv2d, channels_last bf16) on the same conv shapes as
tools/microbench_conv.py / tools/dw_bench.py, next to the engine's own
operator (ssn_op_conv_bf16 / ssn_op_dw_bf16) on identical tensors.

    python tools/cudnn_ref.py [--cases 2,6,8] [--dw]
cuDNN computes the FULL (unsliced) conv of the given widths; the engine reads
the leading slice of a max-shape tensor.  Both are CUDA-event timed over 20
launches after warm-up.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import paper_2312_16733_b200 as ssn  # noqa: E402

CONV = [  # n, h, w, cin, cout, k, stride  (OFA-R50 max subnet layers at bs64 + probes)
    (64, 112, 112, 32, 64, 3, 1),
    (64, 56, 56, 88, 88, 3, 1),
    (64, 14, 14, 360, 360, 3, 1),
    (64, 56, 56, 88, 256, 1, 1),
    (64, 56, 56, 256, 88, 1, 1),
    (64, 14, 14, 360, 1024, 1, 1),
    (64, 7, 7, 720, 720, 3, 1),
    (64, 7, 7, 2048, 720, 1, 1),
    (64, 28, 28, 176, 176, 3, 1),
    (64, 14, 14, 1024, 360, 1, 1),
    (64, 7, 7, 720, 2048, 1, 1),
    (64, 28, 28, 176, 512, 1, 1),
    (64, 28, 28, 512, 176, 1, 1),
    (64, 14, 14, 384, 384, 3, 1),
    (256, 14, 14, 512, 512, 3, 1),
]
DW = [  # n, h, w, c, k, stride (OFA-MBv3 bs256 depthwise layers)
    (256, 56, 56, 192, 3, 1), (256, 56, 56, 192, 7, 1), (256, 112, 112, 24, 3, 1),
    (256, 112, 112, 144, 3, 2), (256, 14, 14, 576, 3, 1), (256, 7, 7, 1152, 7, 1),
]


def timeit(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / it


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="")
    ap.add_argument("--dw", action="store_true")
    a = ap.parse_args()
    torch.backends.cudnn.benchmark = True
    dev = torch.device("cuda:0")
    sel = {int(c) for c in a.cases.split(",")} if a.cases else None
    for ci, (n, h, w, cin, cout, k, st) in enumerate(CONV):
        if sel is not None and ci not in sel:
            continue
        pad = k // 2
        ho, wo = (h + 2 * pad - k) // st + 1, (w + 2 * pad - k) // st + 1
        x = torch.randn(n, h, w, cin, device=dev).to(torch.bfloat16)
        wt = (torch.randn(cout, k, k, cin, device=dev) * 0.05).to(torch.bfloat16)
        xc = x.permute(0, 3, 1, 2)                      # NCHW view of NHWC = channels_last
        wc = wt.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
        t_cudnn = timeit(lambda: F.conv2d(xc, wc, stride=st, padding=pad))
        sc = torch.ones(cout, device=dev)
        sh = torch.zeros(cout, device=dev)
        y = torch.empty(n, ho, wo, cout, device=dev, dtype=torch.bfloat16)
        t_ssn = timeit(lambda: ssn.op_conv_bf16(x, n, h, w, cin, wt, cout, cin, k, st, pad, cout, sc,
                                                sh, None, 1, 0, y))
        fl = 2.0 * n * ho * wo * cout * cin * k * k
        print(f"conv{ci} n{n} {h}x{w} {cin}->{cout} k{k} s{st}: cudnn {t_cudnn:7.1f} us "
              f"({fl / t_cudnn / 1e6:6.0f} TF/s)  ssn {t_ssn:7.1f} us ({fl / t_ssn / 1e6:6.0f} TF/s)",
              flush=True)
    if a.dw:
        for (n, h, w, c, k, st) in DW:
            pad = k // 2
            ho, wo = (h + 2 * pad - k) // st + 1, (w + 2 * pad - k) // st + 1
            x = torch.randn(n, h, w, c, device=dev).to(torch.bfloat16)
            wt = (torch.randn(k, k, c, device=dev) / k).to(torch.bfloat16)
            xc = x.permute(0, 3, 1, 2)
            wc = wt.permute(2, 0, 1).unsqueeze(1).contiguous()
            t_cudnn = timeit(lambda: F.conv2d(xc, wc, stride=st, padding=pad, groups=c))
            sc = torch.ones(c, device=dev)
            sf = torch.zeros(c, device=dev)
            y = torch.empty(n, ho, wo, c, device=dev, dtype=torch.bfloat16)
            s = torch.cuda.current_stream().cuda_stream
            t_ssn = timeit(lambda: ssn.op_dw_bf16(x, n, h, w, c, wt, c, k, k, st, sc, sf, 1, y, s))
            by = 2.0 * (n * h * w * c + n * ho * wo * c)
            print(f"dw n{n} {h}x{w} c{c} k{k} s{st}: cudnn {t_cudnn:7.1f} us ({by / t_cudnn / 1e3:5.0f} GB/s)"
                  f"  ssn {t_ssn:7.1f} us ({by / t_ssn / 1e3:5.0f} GB/s)", flush=True)


if __name__ == "__main__":
    main()
