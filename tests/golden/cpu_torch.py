"""A TUNED torch-CPU baseline of the config-2 workload (test / bench
infrastructure, never the product path).

The oracle port (oracle/ssn_oracle.c) is a direct-convolution restatement: it
is the checker and the reference arm, not a fair CPU speed.  This module runs
the same OFA-ResNet50 subnets through oneDNN (torch.nn.functional.conv2d) the
way a CPU deployment would: each subnet extracted once (leading weight slices
made contiguous, SubnetNorm folded into the conv weights and bias),
channels_last activations, inference mode, every host thread.  Weights come
from make_golden.resnet50 (the ssn_rng.h spec), SubnetNorm rows from one
batch-statistics calibration pass at 32 px (values do not affect speed).
bench.py reports it as ``cpu_baseline_torch`` beside the oracle's
``cpu_baseline``.
"""
import os
import sys
import time

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as G  # noqa: E402

# make_golden pins 8 threads for reproducible fixtures; a baseline uses all of them.
torch.set_num_threads(os.cpu_count() or 1)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2312_16733_b200.supernets import ofa_resnet50_preset  # noqa: E402  (pure Python)


def r50_cfg(name):
    c = ofa_resnet50_preset(name)
    return (c.depth_flags, c.expand_ratios, c.width_multipliers)


class Extracted(G.Run):
    """One subnet, extracted: per conv call site a contiguous channels_last
    weight with the SubnetNorm scale folded in and the shift as conv bias."""

    def __init__(self, net, stats):
        super().__init__(net, False, stats)
        self.cache, self.site = {}, 0

    def conv_bn(self, x, t, n, k, stride, cout, groups=1, res=None, relu=True, res_post=False):
        site, self.site = self.site, self.site + 1
        if site not in self.cache:
            w = self.net.w[t]
            off = (w.shape[2] - k) // 2
            ws = w[:cout, :(x.shape[1] if groups == 1 else w.shape[1]), off:off + k, off:off + k]
            mu = self.stats[0][self.cursor:self.cursor + cout]
            var = self.stats[1][self.cursor:self.cursor + cout]
            self.cursor += cout
            s = self.net.g[n][:cout] / torch.sqrt(var + 1e-5)
            wf = (ws * s[:, None, None, None]).contiguous(memory_format=torch.channels_last)
            self.cache[site] = (wf, self.net.b[n][:cout] - mu * s)
        wf, bias = self.cache[site]
        y = F.conv2d(x, wf, bias, stride=stride, padding=k // 2, groups=groups)
        if res is not None and not res_post:
            y = y + res
        if relu:
            y = torch.relu(y)
        if res is not None and res_post:
            y = y + res
        return y


def extract(fwd, net, cfg):
    r = G.Run(net, True)
    with torch.inference_mode():
        fwd(r, cfg, torch.zeros(2, 3, 32, 32).uniform_())
    return Extracted(net, (torch.cat(r.means), torch.cat(r.vars)))


def r50_sweep(image=224, batch=8, seconds=10.0, subnets=("min", "mid", "max")):
    """images/s of {subnets} x batch per round, rounds until `seconds` pass
    (after one untimed warm-up round that also extracts the subnets)."""
    fwd, net = G.resnet50(0)
    runs = [(s, r50_cfg(s), extract(fwd, net, r50_cfg(s))) for s in subnets]
    x = torch.rand(batch, 3, image, image).contiguous(memory_format=torch.channels_last)

    def one_round():
        for _, cfg, r in runs:
            r.site = 0
            fwd(r, cfg, x)
    with torch.inference_mode():
        one_round()
        n, t0 = 0, time.perf_counter()
        while True:
            one_round()
            n += batch * len(runs)
            el = time.perf_counter() - t0
            if el >= seconds:
                break
    return {"value": round(n / el, 1), "unit": "images/s", "cores": torch.get_num_threads(),
            "kind": "port", "impl": f"torch {torch.__version__} CPU (oneDNN), fp32",
            "sample": f"{n} images: bs{batch} x {{{','.join(subnets)}}} per round at "
                      f"{image}x{image}, subnets extracted (contiguous slices, SubnetNorm "
                      f"folded), channels_last, {el:.1f} s"}


if __name__ == "__main__":
    print(r50_sweep(seconds=float(sys.argv[1]) if len(sys.argv) > 1 else 5.0))
