import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2312_16733_b200 as ssn
for fam_name, B in (("mbv3", 128), ("bert", 64), ("r50", 64)):
    fam = {"r50": ssn.FAMILY_OFA_RESNET50, "mbv3": ssn.FAMILY_OFA_MBV3, "bert": ssn.FAMILY_BERT}[fam_name]
    size = 128 if fam == ssn.FAMILY_BERT else 224
    desc = ssn.make_desc(fam, ssn.DTYPE_BF16, image_size=size, num_classes=2 if fam == ssn.FAMILY_BERT else 1000,
                         max_batch=B, seed=7, input_format=ssn.INPUT_U8_NHWC)
    eng = ssn.Engine(desc)
    for i, n in enumerate(("min", "mid", "max")):
        eng.register_subnet(i, ssn.supernets.preset(fam, n))
    eng.prepare([B])
    rng = np.random.default_rng(7)
    x = rng.integers(0, 30522, size=(B, size), dtype=np.int32) if fam == ssn.FAMILY_BERT else rng.integers(0, 256, size=(B, size, size, 3), dtype=np.uint8)
    res = []
    for it in range(2):
        outs = []
        for i in range(3):
            eng.actuate(i)
            outs.append(eng.infer(x, B, B))
        res.append(outs)
    ok = all(np.array_equal(a, b, equal_nan=True) for a, b in zip(res[0], res[1]))
    print(fam_name, "graph reruns bit-identical:", ok)
    eng.close()
