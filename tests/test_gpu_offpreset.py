"""Off-preset control tuples: widths / expand ratios far below the OFA and
DynaBERT presets, at batch 1-2, where graph-capture-time tiling (chosen from
the MAX shape) meets a much narrower active slice.

Regression for split-K with fewer active K blocks than splits: the split
count is fixed at capture from the max shape, so a narrow subnet can leave a
split with an empty K range (e.g. BERT FFN expand 0.1 -> 304 channels = 5 K
blocks under the 6-way split of the bs1 FFN-down layer; OFA-R50 width 0.1 on
the 7 px 3x3 at bs1).  Such a split must contribute zeros, not hang.

Every case is compared with the CPU oracle (bf16 storage emulated), rel 2e-2.
"""
import numpy as np
import pytest

import paper_2312_16733_b200 as ssn
from oracle import oracle as O
from parity import check_bert

pytestmark = pytest.mark.gpu

SEED = 0


def rel(a, b):
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-12))


def test_bert_ffn_expand_0p1_small_batch(gpu):
    desc = ssn.make_desc(ssn.FAMILY_BERT, ssn.DTYPE_BF16, image_size=128, num_classes=2,
                         max_batch=8, seed=SEED)
    on = O.OracleNet(ssn.FAMILY_BERT, seed=SEED, classes=2, bf16_weights=True)
    cases = [ssn.bert_config(1.0, 1.0, ffn=0.1), ssn.bert_config(0.25, 0.5, ffn=0.1),
             ssn.bert_config(0.1, 1.0, ffn=0.05)]
    with ssn.Engine(desc) as eng:
        for i, c in enumerate(cases):
            eng.register_subnet(i, c)
        eng.prepare([1, 2, 8])
        for i, c in enumerate(cases):
            eng.actuate(i)
            for b in (1, 2):
                ids = O.tokens(SEED, 20 + b, b, 128)
                got = eng.infer(ids, b, b)
                check_bert(f"bert ffn-narrow {i} bs{b}", got, on, c, ids)


R50_NARROW = {
    "w0.1": ssn.SubnetConfig([True] * 9, [0.35] * 18, [0.1] * 6),
    "w0.1_e0.1": ssn.SubnetConfig([True] * 9, [0.1] * 18, [0.1] * 6),
    "w0.3_mixed": ssn.SubnetConfig([False, True, False, True, False, True, True, False, True],
                                   [0.1, 0.35] * 9, [0.3, 1.0, 0.2, 0.5, 0.15, 0.3]),
}


@pytest.mark.parametrize("name", list(R50_NARROW))
def test_r50_narrow_subnets_bs1_224(gpu, name):
    cfg = R50_NARROW[name]
    desc = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, ssn.DTYPE_BF16, image_size=224,
                         num_classes=1000, max_batch=64, seed=SEED)
    on = O.OracleNet(ssn.FAMILY_OFA_RESNET50, seed=SEED, classes=1000, bf16_weights=True)
    x = O.images(SEED, 31, 2, 224)
    m, v = on.calibrate(cfg, O.images(SEED, 130, 8, 224))
    with ssn.Engine(desc) as eng:
        eng.register_subnet(0, cfg, m, v)
        eng.prepare([1, 2, 64])
        eng.actuate(0)
        emu = on.forward(cfg, x, mean=m, var=v, bf16_storage=True)
        for b in (1, 2):
            got = eng.infer(x[:b], b, b)
            assert np.isfinite(got).all()
            assert rel(got, emu[:b]) <= 2e-2, (b, rel(got, emu[:b]))
        # the same images on the bs64 graph (unsplit tiles) agree too
        got64 = eng.infer(x, 2, 64)
        assert rel(got64, emu) <= 2e-2


def test_mbv3_expand1_small_batch(gpu):
    cfg = ssn.SubnetConfig([False, True] * 5, [1.0, 2.0] * 10, [1.0], [3, 7] * 10)
    desc = ssn.make_desc(ssn.FAMILY_OFA_MBV3, ssn.DTYPE_BF16, image_size=224, num_classes=1000,
                         max_batch=8, seed=SEED)
    on = O.OracleNet(ssn.FAMILY_OFA_MBV3, seed=SEED, classes=1000, bf16_weights=True)
    m, v = on.calibrate(cfg, O.images(SEED, 140, 8, 224))
    x = O.images(SEED, 41, 2, 224)
    with ssn.Engine(desc) as eng:
        eng.register_subnet(0, cfg, m, v)
        eng.prepare([1, 2])
        eng.actuate(0)
        emu = on.forward(cfg, x, mean=m, var=v, bf16_storage=True)
        for b in (1, 2):
            got = eng.infer(x[:b], b, b)
            assert np.isfinite(got).all()
            assert rel(got, emu[:b]) <= 2e-2, (b, rel(got, emu[:b]))


def test_forward_on_two_streams_is_ordered(gpu):
    """Forwards of one engine on different streams never overlap (ssn.h)."""
    import torch
    desc = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, ssn.DTYPE_BF16, image_size=64,
                         num_classes=1000, max_batch=16, seed=SEED)
    x = O.images(SEED, 51, 16, 64)
    with ssn.Engine(desc) as eng:
        eng.register_subnet(0, ssn.ofa_resnet50_preset("max"))
        eng.register_subnet(1, ssn.ofa_resnet50_preset("min"))
        eng.prepare([16])
        eng.actuate(0)
        ref0 = eng.infer(x, 16, 16)
        eng.actuate(1)
        ref1 = eng.infer(x, 16, 16)
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        xd = torch.from_numpy(x).cuda()
        out = [np.zeros((16, 1000), np.float32) for _ in range(6)]
        for k in range(6):
            eng.actuate(k % 2)
            eng.forward(xd, 16, 16, out[k], stream=(s1 if k % 3 else s2).cuda_stream)
        torch.cuda.synchronize()
        for k in range(6):
            np.testing.assert_array_equal(out[k], ref0 if k % 2 == 0 else ref1)


def test_register_subnet_rejects_bad_stat_lengths(gpu):
    desc = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, ssn.DTYPE_BF16, image_size=64,
                         num_classes=1000, max_batch=4, seed=SEED)
    cfg = ssn.ofa_resnet50_preset("mid")
    with ssn.Engine(desc) as eng:
        n = eng.stat_count(cfg)
        with pytest.raises(ValueError):
            eng.register_subnet(0, cfg, np.zeros(n - 1, np.float32), np.ones(n - 1, np.float32))
        with pytest.raises(ValueError):
            eng.register_subnet(0, cfg, np.zeros(n, np.float32), None)
        eng.register_subnet(0, cfg, np.zeros(n, np.float32), np.ones(n, np.float32))
