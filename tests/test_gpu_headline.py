"""Oracle parity ON THE BENCHMARKED GRAPHS (BASELINE configs 2, 3, 5).

bench.py times OFA-ResNet50 {min, mid, max} at 224 px on the bs64 CUDA
graphs with uint8 NHWC input and the engine's default SubnetNorm rows,
OFA-MBv3 on the bs256 graphs and BERT on the bs64 graphs.  These tests run
exactly those graphs (same descriptor, same subnet ids, same batch key) and
compare rows with the CPU oracle (oracle/ssn_oracle.c) on the same inputs:

  * every logit finite (all rows of the batch, not only the compared ones);
  * rel L2 <= 2e-2 against the oracle with bf16 activation storage emulated
    AND against the pure-fp32 oracle (north_star: "bf16 rel 2e-2");
  * argmax equal to the bf16-storage oracle on every compared row that is
    not a near tie (top-2 margin <= 4x that row's largest logit error: an
    argmax can only flip when the margin is <= 2x the largest error), and at
    most one near-tie flip in the 8 rows.  The GPU path is bit-reproducible,
    so these counts are deterministic; they are printed.
  * BERT: the measured-floor criterion of tests/parity.py (its bf16-storage
    semantics is implementation-sensitive on these inputs).

The uncalibrated (default-row) random network gives every image the same
argmax (measured), so its argmax check is weak by construction; the
calibrated rows (oracle batch statistics) are the argmax
gate.
"""
import numpy as np
import pytest

import paper_2312_16733_b200 as ssn
from oracle import oracle as O
from parity import check_bert, near_ties

pytestmark = pytest.mark.gpu

SEED = 0
NCMP = 8
REL = 2e-2


def rel(a, b):
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-12))


def u8_to_nchw(u8):
    """INPUT_U8_NHWC semantics (include/ssn.h): value = (u8 - 128) / 64."""
    return ((u8.astype(np.float32) - 128.0) / 64.0).transpose(0, 3, 1, 2).copy()


def argmax_gate(got, ref):
    """Returns (near-tie rows, all argmax flips, flips outside near ties)."""
    near = near_ties(ref, got)
    flip = got.argmax(1) != ref.argmax(1)
    return int(near.sum()), int(flip.sum()), int((flip & ~near).sum())


def check_rows(tag, got_all, emu, ref, calibrated):
    assert np.isfinite(got_all).all(), f"{tag}: non-finite logits in " \
        f"{int((~np.isfinite(got_all)).any(axis=1).sum())} of {len(got_all)} rows"
    got = got_all[:len(ref)]
    e_emu, e_ref = rel(got, emu), rel(got, ref)
    near, flips, bad = argmax_gate(got, emu)
    print(f"{tag}: rel vs bf16-storage oracle {e_emu:.2e}, vs fp32 oracle {e_ref:.2e}, "
          f"argmax flips {flips}/{len(ref)} (outside near ties {bad}; near ties {near}), "
          f"distinct argmax {len(set(emu.argmax(1)))}{' [calibrated]' if calibrated else ''}")
    assert e_emu <= REL, e_emu
    assert e_ref <= REL, e_ref
    assert bad == 0 and flips <= 1


# ------------------------------------------------------------------ config 2
R50_NAMES = ("min", "mid", "max")


@pytest.fixture(scope="module")
def r50_bench(gpu):
    """The bench.py engine: 224 px, uint8 NHWC, max_batch 256, grid {1, 64},
    ids 0-2 = {min, mid, max} with default rows; ids 3-5 calibrated."""
    desc = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, ssn.DTYPE_BF16, image_size=224,
                         num_classes=1000, max_batch=256, seed=SEED,
                         input_format=ssn.INPUT_U8_NHWC)
    eng = ssn.Engine(desc)
    on = O.OracleNet(ssn.FAMILY_OFA_RESNET50, seed=SEED, classes=1000, bf16_weights=True)
    cal = u8_to_nchw(np.random.default_rng(1000).integers(0, 256, (16, 224, 224, 3),
                                                          dtype=np.uint8))
    stats = {}
    for sid, name in enumerate(R50_NAMES):
        cfg = ssn.ofa_resnet50_preset(name)
        eng.register_subnet(sid, cfg)
        m, v = on.calibrate(cfg, cal)
        eng.register_subnet(3 + sid, cfg, m, v)
        stats[name] = (m, v)
    eng.prepare([1, 64])
    x = np.random.default_rng(SEED).integers(0, 256, (64, 224, 224, 3), dtype=np.uint8)
    yield eng, on, stats, x
    eng.close()


@pytest.mark.parametrize("name", R50_NAMES)
def test_r50_224_bs64_default_rows(r50_bench, name):
    """The exact bench workload: default SubnetNorm rows, bs64 graph, 224 px."""
    eng, on, _, x = r50_bench
    sid = R50_NAMES.index(name)
    cfg = ssn.ofa_resnet50_preset(name)
    eng.actuate(sid)
    got = eng.infer(x, 64, 64)
    xs = u8_to_nchw(x[:NCMP])
    emu = on.forward(cfg, xs, subnet_id=sid, bf16_storage=True)
    ref = on.forward(cfg, xs, subnet_id=sid)
    check_rows(f"r50 {name} default bs64", got, emu, ref, calibrated=False)


@pytest.mark.parametrize("name", R50_NAMES)
def test_r50_224_bs64_calibrated_rows(r50_bench, name):
    eng, on, stats, x = r50_bench
    sid = 3 + R50_NAMES.index(name)
    cfg = ssn.ofa_resnet50_preset(name)
    m, v = stats[name]
    eng.actuate(sid)
    got = eng.infer(x, 64, 64)
    xs = u8_to_nchw(x[:NCMP])
    emu = on.forward(cfg, xs, mean=m, var=v, bf16_storage=True)
    ref = on.forward(cfg, xs, mean=m, var=v)
    check_rows(f"r50 {name} calibrated bs64", got, emu, ref, calibrated=True)


def test_r50_224_bs1_graph_matches_oracle(r50_bench):
    """bs1 runs the late-stage convs split-K (conv_finish_kernel)."""
    eng, on, stats, x = r50_bench
    cfg = ssn.ofa_resnet50_preset("max")
    m, v = stats["max"]
    eng.actuate(5)
    got = eng.infer(x[:1], 1, 1)
    emu = on.forward(cfg, u8_to_nchw(x[:1]), mean=m, var=v, bf16_storage=True)
    assert np.isfinite(got).all()
    assert rel(got, emu) <= REL, rel(got, emu)


# ------------------------------------------------------------------ config 3
@pytest.fixture(scope="module")
def mbv3_bench(gpu):
    desc = ssn.make_desc(ssn.FAMILY_OFA_MBV3, ssn.DTYPE_BF16, image_size=224, num_classes=1000,
                         max_batch=256, seed=SEED, input_format=ssn.INPUT_U8_NHWC)
    eng = ssn.Engine(desc)
    on = O.OracleNet(ssn.FAMILY_OFA_MBV3, seed=SEED, classes=1000, bf16_weights=True)
    cal = u8_to_nchw(np.random.default_rng(1001).integers(0, 256, (16, 224, 224, 3),
                                                          dtype=np.uint8))
    stats = {}
    for sid, name in enumerate(R50_NAMES):
        cfg = ssn.supernets.preset(ssn.FAMILY_OFA_MBV3, name)
        eng.register_subnet(sid, cfg)
        m, v = on.calibrate(cfg, cal)
        eng.register_subnet(3 + sid, cfg, m, v)
        stats[name] = (m, v)
    eng.prepare([256])
    x = np.random.default_rng(SEED + 1).integers(0, 256, (NCMP, 224, 224, 3), dtype=np.uint8)
    yield eng, on, stats, x
    eng.close()


@pytest.mark.parametrize("name", R50_NAMES)
@pytest.mark.parametrize("rows", ["default", "calibrated"])
def test_mbv3_224_bs256_graph(mbv3_bench, name, rows):
    """8 live images on the bs256 graph bench.py times (padding rows untouched)."""
    eng, on, stats, x = mbv3_bench
    cfg = ssn.supernets.preset(ssn.FAMILY_OFA_MBV3, name)
    sid = R50_NAMES.index(name)
    xs = u8_to_nchw(x)
    if rows == "default":
        eng.actuate(sid)
        kw = dict(subnet_id=sid)
    else:
        eng.actuate(3 + sid)
        m, v = stats[name]
        kw = dict(mean=m, var=v)
    got = eng.infer(x, NCMP, 256)
    emu = on.forward(cfg, xs, bf16_storage=True, **kw)
    ref = on.forward(cfg, xs, **kw)
    check_rows(f"mbv3 {name} {rows} bs256", got, emu, ref, calibrated=rows == "calibrated")


# ------------------------------------------------------------------ config 5
@pytest.fixture(scope="module")
def bert_bench(gpu):
    desc = ssn.make_desc(ssn.FAMILY_BERT, ssn.DTYPE_BF16, image_size=128, num_classes=2,
                         max_batch=64, seed=SEED, input_format=ssn.INPUT_U8_NHWC)
    eng = ssn.Engine(desc)
    on = O.OracleNet(ssn.FAMILY_BERT, seed=SEED, classes=2, bf16_weights=True)
    for sid, name in enumerate(R50_NAMES):
        eng.register_subnet(sid, ssn.supernets.preset(ssn.FAMILY_BERT, name))
    eng.prepare([64])
    yield eng, on
    eng.close()


@pytest.mark.parametrize("name", R50_NAMES)
def test_bert_seq128_bs64_graph(bert_bench, name):
    eng, on = bert_bench
    cfg = ssn.supernets.preset(ssn.FAMILY_BERT, name)
    ids = O.tokens(SEED, 11, NCMP, 128)
    eng.actuate(R50_NAMES.index(name))
    got = eng.infer(ids, NCMP, 64)
    check_bert(f"bert {name} bs64", got, on, cfg, ids)
