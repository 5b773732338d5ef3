"""Subnet control tuples and plan accounting for the SubNetAct engine.

``SubnetConfig`` mirrors servesim::SubnetConfig (reference
proj/include/servesim/profile.hpp:28-54): depth flags (LayerSelect), expand
ratios and width multipliers (WeightSlice), with the same ``validate`` rules
(profile.hpp:40-53).  ``kernel_sizes`` is this engine's extension for
elastic-kernel supernets.

Family encodings:
  * TinyCNN (config 1): D = 5 flags, E = 3 ratios (per stage), W = 4.
    The reference's ``default_catalog()`` records (profile.hpp:469-507:
    D = 5 x true, E = {3, 4, 6}, W = 4 x mean width) are actuatable as-is.
  * OFA-ResNet50 (config 2): D = 9 per-block LayerSelect flags
    [stem_res, s1b2, s1b3, s2b2, s2b3, s3b4, s3b5, s4b2, s4b3], E = 18 per-block
    expand ratios, W = 6 width multipliers; ``ofa_resnet50_config`` converts
    OFA's (d[5], e[18], w-index[6]) encoding [external].
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Sequence

OFA_R50_WIDTHS = (0.65, 0.8, 1.0)
OFA_R50_EXPANDS = (0.2, 0.25, 0.35)


@dataclass
class SubnetConfig:
    depth_flags: List[bool] = field(default_factory=lambda: [True])
    expand_ratios: List[float] = field(default_factory=lambda: [1.0])
    width_multipliers: List[float] = field(default_factory=lambda: [1.0])
    kernel_sizes: List[int] = field(default_factory=list)

    def mean_width_multiplier(self) -> float:
        """profile.hpp:33-38."""
        if not self.width_multipliers:
            return 1.0
        return sum(self.width_multipliers) / len(self.width_multipliers)

    def validate(self):
        """profile.hpp:40-53 (same messages)."""
        if not self.depth_flags or not self.expand_ratios or not self.width_multipliers:
            raise ValueError("subnet config lists must be non-empty")
        for e in self.expand_ratios:
            if not e > 0.0:
                raise ValueError("expand ratio must be > 0")
        for w in self.width_multipliers:
            if not w > 0.0 or w > 1.0:
                raise ValueError("width multiplier must be in (0,1]")


def tinycnn_config(depth_flags: Sequence[bool], expand_ratios: Sequence[float],
                   width_multipliers: Sequence[float]) -> SubnetConfig:
    return SubnetConfig(list(depth_flags), list(expand_ratios), list(width_multipliers))


# reference default_catalog() (profile.hpp:469-507): id, accuracy, gflops, mean width
DEFAULT_CATALOG_ROWS = [
    ("sub0", 73.82, 0.9, 0.40),
    ("sub1", 76.69, 1.7, 0.50),
    ("sub2", 77.64, 2.6, 0.60),
    ("sub3", 78.25, 3.9, 0.70),
    ("sub4", 79.44, 5.5, 0.85),
    ("sub5", 80.16, 7.5, 1.00),
]


def default_catalog_configs():
    """The reference default catalog's control tuples, in catalog order."""
    return [(rid, acc, SubnetConfig([True] * 5, [3.0, 4.0, 6.0], [w] * 4))
            for rid, acc, _g, w in DEFAULT_CATALOG_ROWS]


def ofa_resnet50_config(d: Sequence[int], e: Sequence[float], w: Sequence[int]) -> SubnetConfig:
    """OFA (d[5] in {0,1,2}, e[18], w-index[6] in {0,1,2}) -> engine SubnetConfig."""
    d = list(d) if len(d) == 5 else [d[0]] * 5
    e = list(e) if len(e) == 18 else [e[0]] * 18
    w = list(w) if len(w) == 6 else [w[0]] * 6
    flags = [d[0] == 2]
    for s in range(4):
        flags += [d[1 + s] >= 1, d[1 + s] >= 2]
    return SubnetConfig(flags, [float(x) for x in e], [OFA_R50_WIDTHS[i] for i in w])


def ofa_resnet50_preset(name: str) -> SubnetConfig:
    """min / mid / max subnets of SURVEY.md §8(d) config 2."""
    idx = {"min": 0, "mid": 1, "max": 2}[name]
    return ofa_resnet50_config([idx] * 5, [OFA_R50_EXPANDS[idx]] * 18, [idx] * 6)


# ---------------------------------------------------------------------------
# plan accounting (algorithmic FLOPs / bytes per image)

OP_KINDS = {0: "input", 1: "conv", 2: "maxpool", 3: "avgpool", 4: "gap", 5: "linear", 6: "se",
            7: "embed", 8: "attn", 9: "layernorm", 10: "token0"}


def plan_ops(desc, cfg: SubnetConfig):
    """Resolved engine plan rows (ssn_plan_ops) as dicts."""
    from . import lib, check, cfg_to_c
    L = lib()
    s, keep = cfg_to_c(cfg)
    n = ctypes.c_uint32()
    check(L.ssn_plan_ops(ctypes.byref(desc), ctypes.byref(s), None, 0, ctypes.byref(n)), "plan_ops")
    from . import OpInfo
    arr = (OpInfo * n.value)()
    check(L.ssn_plan_ops(ctypes.byref(desc), ctypes.byref(s), arr, n.value, ctypes.byref(n)),
          "plan_ops")
    return [{k: getattr(r, k) for k, _ in OpInfo._fields_} for r in arr]


def plan_cost(desc, cfg: SubnetConfig, elem_bytes: int = 2):
    """Per-image algorithmic cost of the active plan.

    flops  = 2 * MACs of every active conv / linear (WeightSlice extents);
    bytes  = each active op reads its input (+ residual) once and writes its
             output once, plus the active weight slice once (per batch: the
             caller divides weight bytes by the batch).
    Returns dict(flops, act_bytes, weight_bytes, per_op=[...]).
    """
    rows = plan_ops(desc, cfg)
    flops = 0
    act_bytes = 0
    w_bytes = 0
    per = []
    for r in rows:
        if not r["active"]:
            per.append(None)  # keep per_op aligned with the plan's op index
            continue
        kind = OP_KINDS[r["kind"]]
        hw_in = r["hin"] * r["win"]
        hw_out = r["hout"] * r["wout"]
        f = b = wb = 0
        if kind in ("conv", "linear"):
            kk = r["k"] * r["k"]
            if r["depthwise"]:
                f = 2 * hw_out * r["cout"] * kk
                wb = r["cout"] * kk * elem_bytes
            else:
                f = 2 * hw_out * r["cout"] * r["cin"] * kk
                wb = r["cout"] * r["cin"] * kk * elem_bytes
            b = (hw_in * r["cin"] + hw_out * r["cout"] * (2 if r["has_residual"] else 1)) * elem_bytes
            if kind == "linear":
                b = hw_in * r["cin"] * elem_bytes + r["cout"] * 4
        elif kind == "input":
            b = hw_in * 3 * 4 + hw_out * r["cout"] * elem_bytes
        elif kind == "se":  # pool read + scale read/write of the activation
            b = 3 * hw_in * r["cin"] * elem_bytes
        elif kind == "attn":  # QK^T and PV over the active heads, per sequence
            f = 2 * 2 * hw_in * hw_in * r["cin"]
            b = 4 * hw_in * r["cin"] * elem_bytes
        elif kind == "embed":
            b = hw_in * 4 + 2 * hw_out * r["cout"] * elem_bytes
        else:
            b = (hw_in * r["cin"] + hw_out * r["cout"]) * elem_bytes
        flops += f
        act_bytes += b
        w_bytes += wb
        row = dict(r)
        row.update(op=kind, flops=f, bytes=b, weight_bytes=wb)
        per.append(row)
    return dict(flops=flops, act_bytes=act_bytes, weight_bytes=w_bytes, per_op=per)


def ofa_mbv3_config(d: Sequence[int], e: Sequence[float], k: Sequence[int]) -> SubnetConfig:
    """OFA-MBv3 (d[5] in {2,3,4}, e[20], ks[20]) -> engine SubnetConfig."""
    d = list(d) if len(d) == 5 else [d[0]] * 5
    flags = []
    for s in range(5):
        flags += [d[s] >= 3, d[s] >= 4]
    e = list(e) if len(e) == 20 else [e[0]] * 20
    k = list(k) if len(k) == 20 else [k[0]] * 20
    return SubnetConfig(flags, [float(x) for x in e], [1.0], [int(x) for x in k])


def ofa_mbv3_preset(name: str) -> SubnetConfig:
    """min (d2 e3 k3) / mid (d3 e4 k5) / max (d4 e6 k7) of SURVEY.md §8(d) config 3."""
    d, e, k = {"min": (2, 3.0, 3), "mid": (3, 4.0, 5), "max": (4, 6.0, 7)}[name]
    return ofa_mbv3_config([d] * 5, [e] * 20, [k] * 20)


def preset(family: int, name: str) -> SubnetConfig:
    if family == 4:
        return {"min": bert_config(0.25, 0.5), "mid": bert_config(0.5, 0.75),
                "max": bert_config(1.0, 1.0)}[name]
    return ofa_mbv3_preset(name) if family == 3 else ofa_resnet50_preset(name)


BERT_DROP = {1.0: (), 0.75: (3, 7, 11), 0.5: (1, 3, 5, 7, 9, 11)}


def bert_config(mw: float = 1.0, md: float = 1.0, ffn: float = None) -> SubnetConfig:
    """DynaBERT-style (width mw, depth md) -> 12 layer flags, E = [FFN width],
    W = [head width] (depth 0.75 drops layers 3/7/11, 0.5 the
    odd layers)."""
    drop = BERT_DROP[md]
    return SubnetConfig([i not in drop for i in range(12)], [ffn if ffn else mw], [mw])
