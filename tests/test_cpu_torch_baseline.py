"""The tuned torch-CPU baseline (tests/golden/cpu_torch.py, bench.py
``cpu_baseline_torch``) computes the same subnet as the golden restatement:
extracting a subnet (contiguous slices, SubnetNorm folded into the conv) must
not change its logits."""
import os
import sys

import pytest
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import cpu_torch as C  # noqa: E402
import make_golden as G  # noqa: E402


@pytest.mark.parametrize("name", ["min", "mid", "max"])
def test_extracted_subnet_matches_restatement(name):
    fwd, net = G.resnet50(0)
    cfg = C.r50_cfg(name)
    ext = C.extract(fwd, net, cfg)
    x = torch.rand(2, 3, 32, 32, generator=torch.Generator().manual_seed(1))
    with torch.inference_mode():
        a = fwd(ext, cfg, x.contiguous(memory_format=torch.channels_last))
        b = fwd(G.Run(net, False, ext.stats), cfg, x)
    assert float((a - b).norm() / b.norm()) < 1e-4


def test_sweep_reports_contract_fields():
    r = C.r50_sweep(image=32, batch=2, seconds=0.05, subnets=("min",))
    assert r["value"] > 0 and r["unit"] == "images/s" and r["cores"] >= 1
    assert r["kind"] == "port" and "sample" in r
