"""CPU tests of the subnet-selection side (config 4), against the UNMODIFIED
reference compiled into oracle/_ref/servesim_ref:
  * the reference binary reproduces the frozen SlackFit decisions of
    test_policy.cpp:83-127 (pins the oracle itself);
  * catalog CSVs written by the engine's profiler are accepted by the
    reference's parse_catalog_csv (P1 check, profile.hpp:392-444) and drive
    its simulator; every dispatch targets a profiled (subnet, batch) that the
    engine can actuate and run (graph key = profiled_batch, policy.hpp:219-232).
"""
import json
import os
import subprocess

import pytest

from oracle import oracle as O
from paper_2312_16733_b200 import profiler

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_reference_frozen_slackfit_decisions():
    got = O.ref_decide("default", 20, [36000, 23000, 15000, 12500, 9000, 4000, 3000, 2000, -5000])
    assert got == [(32, 5, 24000), (64, 4, 16800), (32, 3, 12500), (64, 2, 11900),
                   (64, 0, 7600), (8, 0, 3900), None, None, None]


def fake_rows():
    base = [300, 420, 480, 560, 700, 900]
    rows = []
    for i, (sid, acc, _cfg) in enumerate(profiler.b200_r50_catalog()):
        prev = 0
        for b in profiler.REFERENCE_BATCHES:
            us = max(int(base[i] * (1 + 0.04 * b)), prev + 1)
            prev = us
            rows.append((sid, acc, 1.0 + i, b, us))
    return rows


def test_profiler_csv_drives_reference_simulator(tmp_path):
    rows = fake_rows()
    csv_path = str(tmp_path / "cat.csv")
    profiler.write_catalog_csv(rows, csv_path)
    assert profiler.read_catalog_csv(csv_path) == rows
    assert profiler.holds_p1_p2(rows) == (True, True)
    trace = str(tmp_path / "t.jsonl")
    subprocess.run([O.REF_BIN, "gen-trace", "800", "3200", "4", "1", "6000", "3", trace], check=True)
    log = str(tmp_path / "log.tsv")
    out = subprocess.run([O.REF_BIN, "simulate", csv_path, trace, "2", "0", "slackfit", log],
                         check=True, capture_output=True, text=True).stdout
    rep = json.loads(out)
    assert rep["total"] > 0
    grid = set(profiler.REFERENCE_BATCHES)
    with open(log) as f:
        recs = [line.split("\t") for line in f]
    assert recs
    for r in recs:
        subnet, count, batch = int(r[3]), int(r[4]), int(r[5])
        assert 0 <= subnet < 6 and batch in grid and 1 <= count <= batch


def test_reference_rejects_p1_violation(tmp_path):
    rows = fake_rows()
    bad = [list(r) for r in rows]
    bad[3][4] = bad[2][4]  # l(8) == l(4)
    csv_path = str(tmp_path / "bad.csv")
    profiler.write_catalog_csv(bad, csv_path)
    r = subprocess.run([O.REF_BIN, "decide", csv_path, "20", "1000"], capture_output=True, text=True)
    assert r.returncode == 2 and "violates latency monotonicity" in r.stderr
