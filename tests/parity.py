"""Shared parity criteria for the GPU tests (test infrastructure).

BERT (config 5) needs a measured tolerance.  Its bf16-storage semantics is
not a unique function: changing ONLY the fp32 accumulation order of the
linears (oracle acc64 flag) moves the bf16-stored network's 2-class logits by
0.6-2.5% on the test inputs, while the same change moves the pure-fp32
network by ~1e-6 (tests/test_cpu_oracle.py::test_bert_bf16_storage_is_
implementation_sensitive) — bf16 rounding-boundary flips are amplified over
12 post-LN layers.  So the GPU (fp32 tensor-core accumulation in its own
order) is held to

  rel(GPU, bf16-storage oracle) <= max(2e-2, 1.5 x rel(oracle acc32, oracle acc64))
  rel(GPU, fp32 oracle)         <= max(2e-2, 1.5 x rel(bf16-storage oracle, fp32 oracle))

both floors measured on the SAME inputs, plus argmax equality with the fp32
oracle on every row that is not a near tie.
"""
import numpy as np

REL = 2e-2


def rel(a, b):
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-12))


def near_ties(ref, got):
    top2 = np.sort(ref, axis=1)[:, -2:]
    margin = top2[:, 1] - top2[:, 0]
    return margin <= 4.0 * np.abs(got - ref).max(axis=1)


def check_bert(tag, got, on, cfg, ids):
    emu = on.forward_tokens(cfg, ids, bf16_storage=True)
    emu64 = on.forward_tokens(cfg, ids, bf16_storage=True, acc64=True)
    ref = on.forward_tokens(cfg, ids)
    impl_floor, bf16_floor = rel(emu64, emu), rel(emu, ref)
    tol_emu, tol_ref = max(REL, 1.5 * impl_floor), max(REL, 1.5 * bf16_floor)
    e_emu, e_ref = rel(got, emu), rel(got, ref)
    near = near_ties(ref, got)
    bad = int(((got.argmax(1) != ref.argmax(1)) & ~near).sum())
    print(f"{tag}: rel vs bf16-storage oracle {e_emu:.2e} (tol {tol_emu:.2e}; acc32/acc64 "
          f"floor {impl_floor:.2e}), vs fp32 oracle {e_ref:.2e} (tol {tol_ref:.2e}; bf16 floor "
          f"{bf16_floor:.2e}), argmax mismatches {bad} (near ties {int(near.sum())})")
    assert np.isfinite(got).all()
    assert e_emu <= tol_emu, (e_emu, tol_emu)
    assert e_ref <= tol_ref, (e_ref, tol_ref)
    assert bad == 0
    return e_emu, e_ref
