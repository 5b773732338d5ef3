"""§8f on the GPU through the C++ harness tools/_bin/serve_live (compiled
against the UNMODIFIED reference headers, include/ssn_serve.hpp):

  * the profiler writes a catalog CSV the reference parser accepts
    (parse_catalog_csv, P1 enforced, profile.hpp:392-444) with P2 holding,
    and the reference's own SlackFit (oracle/_ref/servesim_ref) decides on it;
  * engine-backed live serving (the sleep of serve_runtime.hpp:167 replaced
    by ssn_actuate + ssn_forward) tracks the reference simulator on the same
    bursty trace (acceptance.cpp:429-452: |d attainment| <= 0.02,
    |d accuracy| <= 0.5), and the first dispatch's logits (EngineWorker ->
    unmodified serve_detail::DispatchCmd) match the CPU oracle.
"""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2312_16733_b200 as ssn
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "_bin", "serve_live")


def run(*args, timeout=600):
    out = subprocess.run([EXE, *map(str, args)], check=True, capture_output=True, text=True,
                         timeout=timeout).stdout
    return json.loads(out.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def catalog(gpu, tmp_path_factory):
    if not os.path.exists(EXE):
        pytest.fail("tools/_bin/serve_live missing (built by __graft_entry__.build())")
    path = str(tmp_path_factory.mktemp("cat") / "catalog_b200.csv")
    rep = run("profile", "--out", path, "--iters", "10")
    return path, rep


def test_profiler_csv_loads_through_reference_parser(catalog):
    path, rep = catalog
    assert rep["p1"] and rep["p2"], rep
    assert rep["subnets"] == 6 and rep["batches"] == [1, 2, 4, 8, 16, 32, 64]
    lat = {(r["subnet"], r["batch"]): r["latency_us"] for r in rep["rows"]}
    assert all(lat[(s, 1)] < lat[(s, 64)] for s in ("sub0", "sub5"))
    # the reference's SlackFit decides on the B200 profile (policy.hpp:191)
    if O.ref_available():
        d = O.ref_decide(path, 20, [lat[("sub0", 1)] + 1, lat[("sub5", 64)] + 1, 10 ** 6])
        assert d[0] is not None and d[0][1] == 0       # tightest slack: sub0
        assert d[-1] is not None and d[-1][1] == 5      # unconstrained: most accurate


def test_live_engine_workers_track_the_simulator(catalog, tmp_path):
    path, _ = catalog
    dump = str(tmp_path / "first.bin")
    rep = run("serve", "--catalog", path, "--workers", 1, "--seeds", 21, "--duration", 3,
              "--load", 0.3, "--dump-first", dump)
    r = rep["runs"][0]
    print(json.dumps({k: r[k] for k in ("d_attainment", "d_accuracy", "dispatches",
                                        "subnet_switches", "served_img_s_wall",
                                        "service_over_profiled")}))
    assert r["live"]["total"] == r["queries"] > 1000
    assert r["criterion12_pass"], r
    # EngineWorker's first dispatch: logits vs the oracle on the same images
    raw = open(dump, "rb").read()
    off, count, subnet, row = (int(v) for v in np.frombuffer(raw[:16], np.uint32))
    img = 224 * 224 * 3
    u8 = np.frombuffer(raw[16:16 + count * img], np.uint8).reshape(count, 224, 224, 3)
    got = np.frombuffer(raw[16 + count * img:], np.float32).reshape(count, 1000)
    from paper_2312_16733_b200 import profiler
    cfg = profiler.b200_r50_catalog()[row][2]   # default SubnetNorm rows of engine id `subnet`
    on = O.OracleNet(ssn.FAMILY_OFA_RESNET50, seed=0, classes=1000, bf16_weights=True)
    k = min(count, 4)
    x = ((u8[:k].astype(np.float32) - 128.0) / 64.0).transpose(0, 3, 1, 2).copy()
    emu = on.forward(cfg, x, subnet_id=subnet, bf16_storage=True)
    err = float(np.linalg.norm(got[:k] - emu) / np.linalg.norm(emu))
    assert np.isfinite(got).all() and err <= 2e-2, err
