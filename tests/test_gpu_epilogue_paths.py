"""Alternative code paths compute the SAME bits:

* the TMA-store epilogue (default) vs the padded-fp32-transpose epilogue
  (SSN_TC_DEBUG=33554432): identical per-element math (SubnetNorm FMA,
  residual add, activation, round-to-nearest bf16 — ReLU fused into the
  rounding is exact);
* two K blocks per ring stage (default, >= 16 K blocks) vs one
  (SSN_TC_KPS2_NK=0): the MMAs accumulate the K blocks in the same order;
* the SubnetNorm row staged in shared memory vs warp shuffles
  (SSN_TC_DEBUG=134217728);
* one whole-forward CUDA graph per LayerSelect variant vector (default) vs
  one graph per segment (SSN_NO_FWD_GRAPH=1): the same kernels in the same
  order.

Each setting runs in a fresh process (the engine reads the switches once):
OFA-ResNet50 mid at 64 px bs16 (stage 1-4 1x1 / 3x3 convs, residual ring),
OFA-MBv3 mid (h_swish epilogues) and BERT mid (GELU, residuals from global
memory); logits must match the default run bit for bit.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2312_16733_b200 as ssn
from oracle import oracle as O
out = {{}}
for fam, hw, classes in ((ssn.FAMILY_OFA_RESNET50, 64, 1000), (ssn.FAMILY_OFA_MBV3, 64, 1000),
                         (ssn.FAMILY_BERT, 128, 8)):
    desc = ssn.make_desc(fam, ssn.DTYPE_BF16, image_size=hw, num_classes=classes, max_batch=16, seed=0)
    with ssn.Engine(desc, device=0) as eng:
        eng.register_subnet(0, ssn.supernets.preset(fam, "mid"))
        eng.prepare([16])
        eng.actuate(0)
        x = O.tokens(0, 3, 16, hw) if fam == ssn.FAMILY_BERT else O.images(0, 1, 16, hw)
        out[str(fam)] = eng.infer(x, 16, 16)
np.savez({path!r}, **out)
"""


def _run(tmp_dir, tag, env):
    path = str(tmp_dir / f"{tag}.npz")
    res = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, path=path)], cwd=ROOT,
                         env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    return np.load(path)


@pytest.fixture(scope="module")
def default_logits(gpu, tmp_path_factory):
    return _run(tmp_path_factory.mktemp("epi"), "default", {"SSN_TC_DEBUG": "0"})


@pytest.mark.parametrize("tag,env", [
    ("transpose_epilogue", {"SSN_TC_DEBUG": "33554432"}),
    ("one_k_block_per_stage", {"SSN_TC_KPS2_NK": "0"}),
    ("shuffled_subnetnorm", {"SSN_TC_DEBUG": "134217728"}),
    ("segment_graphs", {"SSN_NO_FWD_GRAPH": "1"}),
])
def test_conv_tc_paths_bitwise_equal(default_logits, tmp_path, tag, env):
    base = default_logits
    alt = _run(tmp_path, tag, env)
    for fam in base.files:
        a, b = base[fam], alt[fam]
        assert np.isfinite(a).all()
        diff = int(np.count_nonzero(a.view(np.uint32) != b.view(np.uint32)))
        print(f"{tag}: family {fam}: {diff} of {a.size} logits differ")
        assert diff == 0
