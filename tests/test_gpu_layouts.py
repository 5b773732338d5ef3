"""Storage-layout switches, each in a fresh process (the engine reads them once):

* SSN_PAD_ROWS=1 / 0 — every bf16 CNN activation row padded to a 16-channel
                     multiple / none (the default pads rows of >= 256
                     channels); every kernel addresses activations through
                     the descriptor row's ldi / ldo (engine.cu act_ld);
* SSN_PACK_WEIGHTS=1 — compact weight rows instead of the default 32-B rows
                     (supernet.hpp Builder::pad16).

Both must give the same oracle parity as the default layout: OFA-ResNet50 mid
and OFA-MBv3 mid (widths 56 / 104 / 408 and 72 / 136 / 408: rows = 8 mod 16)
at 64 px, bs8, rel L2 <= 2e-2 against the bf16-storage oracle.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2312_16733_b200 as ssn
from oracle import oracle as O
worst = 0.0
for fam in (ssn.FAMILY_OFA_RESNET50, ssn.FAMILY_OFA_MBV3):
    hw = 64
    desc = ssn.make_desc(fam, ssn.DTYPE_BF16, image_size=hw, num_classes=1000, max_batch=8, seed=0)
    cfg = ssn.supernets.preset(fam, "mid")
    on = O.OracleNet(fam, seed=0, classes=1000, bf16_weights=True)
    mean, var = on.calibrate(cfg, O.images(0, 100, 8, hw))
    x = O.images(0, 1, 8, hw)
    with ssn.Engine(desc, device=0) as eng:
        eng.register_subnet(0, cfg, mean, var)
        eng.prepare([8])
        eng.actuate(0)
        got = eng.infer(x, 8, 8)
    ref = on.forward(cfg, x, mean=mean, var=var, bf16_storage=True)
    assert np.isfinite(got).all()
    worst = max(worst, float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
print("REL", worst)
"""


@pytest.mark.parametrize("env,val", [("SSN_PAD_ROWS", "1"), ("SSN_PAD_ROWS", "0"),
                                     ("SSN_PACK_WEIGHTS", "1")])
def test_layout_switch_keeps_parity(gpu, env, val):
    out = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)], cwd=ROOT,
                         env={**os.environ, env: val}, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    rel = float([l for l in out.stdout.splitlines() if l.startswith("REL")][-1].split()[1])
    print(f"{env}={val}: worst rel L2 vs bf16-storage oracle {rel:.2e}")
    assert rel <= 2e-2
