"""CPU tests of the drop-in boundary: libssn.so loads, exports every entry
point include/ssn.h declares, its host-only calls work without a GPU, and on
a machine without a B200 the engine fails loudly instead of falling back."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2312_16733_b200 as ssn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ssn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ssn_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 15
    lib = ctypes.CDLL(ssn.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_mirror_binds_every_symbol():
    L = ssn.lib()
    for s in declared_symbols():
        assert getattr(L, s).argtypes is not None or getattr(L, s).restype is not None, s


def test_host_only_calls_without_gpu():
    d = ssn.make_desc(ssn.FAMILY_TINYCNN, ssn.DTYPE_F32, image_size=32, num_classes=10)
    n = ssn.weight_blob_bytes(d)
    blob = ssn.generate_weight_blob(d)
    assert blob.nbytes == n and np.any(blob)
    cfg = ssn.default_catalog_configs()[2][2]
    assert ssn.plan_stat_count(d, cfg) > 0
    ops = ssn.plan_ops(d, cfg)
    assert ops[0]["kind"] == 0 and ops[-1]["kind"] == 5


def test_error_codes_and_last_error():
    L = ssn.lib()
    n = ctypes.c_uint64()
    rc = L.ssn_weight_blob_bytes(None, ctypes.byref(n))
    assert rc == ssn.SSN_E_INVALID
    assert b"null supernet descriptor" in L.ssn_last_error()


def test_engine_refuses_to_run_without_a_b200():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    d = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, image_size=32, max_batch=1)
    with pytest.raises(RuntimeError):
        ssn.Engine(d)


def test_catalog_configs_mirror_reference_default_catalog():
    # profile.hpp:469-507: six subnets, D = 5 x true, E = {3,4,6}, W = 4 x mean width
    rows = ssn.default_catalog_configs()
    assert [r[0] for r in rows] == ["sub0", "sub1", "sub2", "sub3", "sub4", "sub5"]
    assert [r[1] for r in rows] == [73.82, 76.69, 77.64, 78.25, 79.44, 80.16]
    for _, _, c in rows:
        assert c.depth_flags == [True] * 5 and c.expand_ratios == [3.0, 4.0, 6.0]
        assert len(set(c.width_multipliers)) == 1


def test_ofa_encoding_to_layerselect_flags():
    c = ssn.ofa_resnet50_config([2, 0, 1, 2, 1], [0.25] * 18, [2, 1, 0, 2, 1, 0])
    assert c.depth_flags == [True, False, False, True, False, True, True, True, False]
    assert c.width_multipliers == [1.0, 0.8, 0.65, 1.0, 0.8, 0.65]


def test_cpp_binding_against_reference_headers(tmp_path):
    """include/ssn.hpp compiles with the unmodified servesim headers and the
    reference's default_catalog() tuples are actuatable (host-side check)."""
    import shutil
    import subprocess
    ref = "/root/reference/proj/include"
    if not os.path.isdir(ref) or not shutil.which("g++"):
        pytest.skip("reference headers not present")
    exe = tmp_path / "binding"
    inc_json = os.path.join(ROOT, "oracle", "_ref", "inc")
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", f"-I{ref}", f"-I{inc_json}",
                    os.path.join(ROOT, "tests", "cpp", "servesim_binding.cpp"),
                    f"-L{os.path.dirname(ssn.LIB_PATH)}", "-lssn",
                    f"-Wl,-rpath,{os.path.dirname(ssn.LIB_PATH)}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    counts = [int(line.split()[1]) for line in out.splitlines() if line.startswith("sub")]
    assert len(counts) == 6 and counts == sorted(counts)
    assert "invalid_argument: width multiplier must be in (0,1]" in out
