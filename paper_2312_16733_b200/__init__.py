"""B200-native SubNetAct execution engine (Python host mirror over the C-ABI).

The product is ``libssn.so`` (CUDA sm_100a + C++ host code) behind the C-ABI
of ``include/ssn.h``.  This module is a thin ctypes mirror of that ABI so the
tests and ``bench.py`` read like the reference's worker code: a worker
actuates a subnet (``Engine.actuate``) and runs a batch (``Engine.forward``)
where the reference's mock worker sleeps (reference
proj/include/servesim/serve_runtime.hpp:161-172).

Errors mirror the reference's exception types (profile.hpp:40-53,
policy.hpp:92-98): ``ValueError`` for std::invalid_argument, ``IndexError``
for std::out_of_range, ``RuntimeError`` for CUDA failures and call-order
violations.  There is no fallback: if ``libssn.so`` is missing or fails to
load, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

from .supernets import (  # noqa: F401  (re-exported)
    SubnetConfig,
    default_catalog_configs,
    ofa_resnet50_config,
    ofa_resnet50_preset,
    bert_config,
    plan_cost,
    plan_ops,
    tinycnn_config,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libssn.so")

FAMILY_TINYCNN = 1
FAMILY_OFA_RESNET50 = 2
FAMILY_OFA_MBV3 = 3
FAMILY_BERT = 4
DTYPE_F32 = 0
DTYPE_BF16 = 1
INPUT_F32_NCHW = 0
INPUT_U8_NHWC = 1

SSN_OK = 0
SSN_E_INVALID = -1
SSN_E_RANGE = -2
SSN_E_CUDA = -3
SSN_E_STATE = -4
SSN_E_NOMEM = -5


class SupernetDesc(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_uint32),
        ("dtype", ctypes.c_uint32),
        ("image_size", ctypes.c_uint32),
        ("num_classes", ctypes.c_uint32),
        ("max_batch", ctypes.c_uint32),
        ("input_format", ctypes.c_uint32),
        ("seed", ctypes.c_uint64),
        ("reserved", ctypes.c_uint32 * 8),
    ]


class _SubnetCfgC(ctypes.Structure):
    _fields_ = [
        ("depth_flags", ctypes.POINTER(ctypes.c_uint8)),
        ("n_depth", ctypes.c_uint32),
        ("expand_ratios", ctypes.POINTER(ctypes.c_double)),
        ("n_expand", ctypes.c_uint32),
        ("width_multipliers", ctypes.POINTER(ctypes.c_double)),
        ("n_width", ctypes.c_uint32),
        ("kernel_sizes", ctypes.POINTER(ctypes.c_uint32)),
        ("n_kernel", ctypes.c_uint32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("weight_bytes", ctypes.c_uint64),
        ("norm_table_bytes", ctypes.c_uint64),
        ("max_subnet_stat_bytes", ctypes.c_uint64),
        ("arena_bytes", ctypes.c_uint64),
        ("registered_subnets", ctypes.c_uint32),
        ("active_subnet", ctypes.c_int32),
        ("graphs_built", ctypes.c_uint32),
        ("last_forward_kernels", ctypes.c_uint32),
        ("last_forward_graphs", ctypes.c_uint32),
        ("reserved0", ctypes.c_uint32),
        ("last_actuate_us", ctypes.c_double),
        ("last_forward_host_us", ctypes.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved0"}


class OpInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in (
        "kind", "active", "k", "stride", "hin", "win", "hout", "wout", "cin", "cout",
        "cin_max", "cout_max", "depthwise", "segment", "block", "has_residual")]


def cfg_to_c(cfg: SubnetConfig):
    """Marshal a SubnetConfig; returns (struct, keepalive)."""
    d = (ctypes.c_uint8 * len(cfg.depth_flags))(*[1 if f else 0 for f in cfg.depth_flags])
    e = (ctypes.c_double * len(cfg.expand_ratios))(*cfg.expand_ratios)
    w = (ctypes.c_double * len(cfg.width_multipliers))(*cfg.width_multipliers)
    k = (ctypes.c_uint32 * max(1, len(cfg.kernel_sizes)))(*cfg.kernel_sizes)
    s = _SubnetCfgC(
        ctypes.cast(d, ctypes.POINTER(ctypes.c_uint8)), len(cfg.depth_flags),
        ctypes.cast(e, ctypes.POINTER(ctypes.c_double)), len(cfg.expand_ratios),
        ctypes.cast(w, ctypes.POINTER(ctypes.c_double)), len(cfg.width_multipliers),
        ctypes.cast(k, ctypes.POINTER(ctypes.c_uint32)) if cfg.kernel_sizes else None,
        len(cfg.kernel_sizes),
    )
    return s, (d, e, w, k)


_lib_handle = None


def lib() -> ctypes.CDLL:
    """Load libssn.so (raises if absent — there is no fallback path)."""
    global _lib_handle
    if _lib_handle is not None:
        return _lib_handle
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"SubNetAct engine library missing: {LIB_PATH} (run `python __graft_entry__.py build`)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    u32, u64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    desc_p = ctypes.POINTER(SupernetDesc)
    cfg_p = ctypes.POINTER(_SubnetCfgC)
    fp = ctypes.POINTER(ctypes.c_float)
    sig = {
        "ssn_weight_blob_bytes": (i32, [desc_p, ctypes.POINTER(u64)]),
        "ssn_generate_weight_blob": (i32, [desc_p, P, u64]),
        "ssn_plan_stat_count": (i32, [desc_p, cfg_p, ctypes.POINTER(u64)]),
        "ssn_plan_ops": (i32, [desc_p, cfg_p, P, u32, ctypes.POINTER(u32)]),
        "ssn_create": (i32, [i32, desc_p, P, u64, ctypes.POINTER(P)]),
        "ssn_destroy": (None, [P]),
        "ssn_subnet_stat_count": (i32, [P, cfg_p, ctypes.POINTER(u64)]),
        "ssn_register_subnet": (i32, [P, u32, cfg_p, fp, fp]),
        "ssn_register_subnet_n": (i32, [P, u32, cfg_p, fp, fp, u64]),
        "ssn_prepare": (i32, [P, ctypes.POINTER(u32), u32]),
        "ssn_actuate": (i32, [P, u32]),
        "ssn_forward": (i32, [P, P, u32, u32, P, P]),
        "ssn_synchronize": (i32, [P, P]),
        "ssn_profile_latency": (i32, [P, u32, u32, u32, ctypes.POINTER(ctypes.c_double)]),
        "ssn_profile_ops": (i32, [P, u32, u32, u32, P, u32]),
        "ssn_debug_op_checksums": (i32, [P, u32, u32, P, u32]),
        "ssn_query": (i32, [P, ctypes.POINTER(Stats)]),
        "ssn_device_logits": (i32, [P, ctypes.POINTER(P)]),
        "ssn_last_error": (ctypes.c_char_p, []),
        "ssn_op_conv_bf16": (i32, [P, i32, i32, i32, i32, P, i32, i32, i32, i32, i32, i32,
                                   P, P, P, i32, i32, P, P]),
        "ssn_op_dw_bf16": (i32, [P, i32, i32, i32, i32, P, i32, i32, i32, i32, P, P, i32, P, P]),
        "ssn_op_conv_f32": (i32, [P, i32, i32, i32, i32, P, i32, i32, i32, i32, i32, i32, i32,
                                  i32, P, P, P, i32, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib_handle = L
    return L


def check(rc: int, what: str = ""):
    if rc == SSN_OK:
        return
    msg = lib().ssn_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == SSN_E_INVALID:
        raise ValueError(text)
    if rc == SSN_E_RANGE:
        raise IndexError(text)
    raise RuntimeError(f"[ssn {rc}] {text}")


def make_desc(family: int, dtype: int = DTYPE_BF16, image_size: int = 224, num_classes: int = 1000,
              max_batch: int = 64, seed: int = 0, input_format: int = INPUT_F32_NCHW) -> SupernetDesc:
    d = SupernetDesc()
    d.family, d.dtype, d.image_size = family, dtype, image_size
    d.num_classes, d.max_batch, d.input_format, d.seed = num_classes, max_batch, input_format, seed
    return d


def weight_blob_bytes(desc: SupernetDesc) -> int:
    n = ctypes.c_uint64()
    check(lib().ssn_weight_blob_bytes(ctypes.byref(desc), ctypes.byref(n)), "weight_blob_bytes")
    return n.value


def generate_weight_blob(desc: SupernetDesc):
    """Host weight blob as a numpy uint8 array."""
    import numpy as np
    n = weight_blob_bytes(desc)
    blob = np.zeros(n, dtype=np.uint8)
    check(lib().ssn_generate_weight_blob(ctypes.byref(desc), blob.ctypes.data, n), "generate")
    return blob


def plan_stat_count(desc: SupernetDesc, cfg: SubnetConfig) -> int:
    s, keep = cfg_to_c(cfg)
    n = ctypes.c_uint64()
    check(lib().ssn_plan_stat_count(ctypes.byref(desc), ctypes.byref(s), ctypes.byref(n)),
          "plan_stat_count")
    return n.value


def _ptr(x) -> Optional[int]:
    """Address of a numpy array / torch tensor / int (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(f"unsupported buffer type {type(x)}")


class Engine:
    """One SubNetAct engine = one supernet replica on one GPU."""

    def __init__(self, desc: SupernetDesc, device: int = 0, weights=None):
        self.desc = desc
        self.device = device
        L = lib()
        h = ctypes.c_void_p()
        nbytes = 0 if weights is None else int(weights.nbytes)
        check(L.ssn_create(device, ctypes.byref(desc), _ptr(weights), nbytes, ctypes.byref(h)),
              "ssn_create")
        self._h = h
        self.num_classes = desc.num_classes

    def close(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value and _lib_handle is not None:
                _lib_handle.ssn_destroy(h)
            self._h = None
        except Exception:  # interpreter shutdown: module globals already torn down
            pass

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def stat_count(self, cfg: SubnetConfig) -> int:
        s, keep = cfg_to_c(cfg)
        n = ctypes.c_uint64()
        check(lib().ssn_subnet_stat_count(self._h, ctypes.byref(s), ctypes.byref(n)), "stat_count")
        return n.value

    def register_subnet(self, subnet_id: int, cfg: SubnetConfig, bn_mean=None, bn_var=None):
        import numpy as np
        s, keep = cfg_to_c(cfg)
        fp = ctypes.POINTER(ctypes.c_float)
        m = v = None
        n = 0
        if (bn_mean is None) != (bn_var is None):
            raise ValueError("SubnetNorm statistics need both bn_mean and bn_var (or neither)")
        if bn_mean is not None:
            bn_mean = np.ascontiguousarray(bn_mean, dtype=np.float32)
            bn_var = np.ascontiguousarray(bn_var, dtype=np.float32)
            if bn_mean.ndim != 1 or bn_var.shape != bn_mean.shape:
                raise ValueError("bn_mean / bn_var must be 1-D arrays of equal length")
            n = bn_mean.size
            m = bn_mean.ctypes.data_as(fp)
            v = bn_var.ctypes.data_as(fp)
        # the length-checked entry point: a short array is an error, never a heap over-read
        check(lib().ssn_register_subnet_n(self._h, subnet_id, ctypes.byref(s), m, v, n),
              f"register_subnet({subnet_id})")

    def prepare(self, batch_grid: Sequence[int]):
        arr = (ctypes.c_uint32 * len(batch_grid))(*batch_grid)
        check(lib().ssn_prepare(self._h, arr, len(batch_grid)), "prepare")

    def actuate(self, subnet_id: int):
        check(lib().ssn_actuate(self._h, subnet_id), f"actuate({subnet_id})")

    def forward(self, x, count: int, profiled_batch: int, logits=None, stream=None):
        """Enqueue a forward; `x`/`logits` are host (numpy) or device (torch) buffers."""
        check(lib().ssn_forward(self._h, _ptr(x), count, profiled_batch, _ptr(logits),
                                _ptr(stream)), "forward")

    def synchronize(self, stream=None):
        check(lib().ssn_synchronize(self._h, _ptr(stream)), "synchronize")

    def infer(self, x, count: int, profiled_batch: int):
        """Blocking forward returning numpy float32 logits [count][classes]."""
        import numpy as np
        out = np.zeros((count, self.num_classes), dtype=np.float32)
        self.forward(x, count, profiled_batch, out)
        self.synchronize()
        return out

    def profile_latency(self, subnet_id: int, batch: int, iters: int = 20) -> float:
        us = ctypes.c_double()
        check(lib().ssn_profile_latency(self._h, subnet_id, batch, iters, ctypes.byref(us)),
              "profile_latency")
        return us.value

    def profile_ops(self, subnet_id: int, batch: int, iters: int = 5):
        """Per-op median device µs (ssn_plan_ops order; 0 = skipped op)."""
        import numpy as np
        out = np.zeros(512, dtype=np.float32)
        check(lib().ssn_profile_ops(self._h, subnet_id, batch, iters, out.ctypes.data, 512),
              "profile_ops")
        return out

    def debug_op_checksums(self, subnet_id: int, batch: int):
        """Debugging: per-op FNV-1a hash of every op's output (op-by-op run
        on the last staged input; 0 = op not run)."""
        import numpy as np
        out = np.zeros(512, dtype=np.uint64)
        check(lib().ssn_debug_op_checksums(self._h, subnet_id, batch, out.ctypes.data, 512),
              "debug_op_checksums")
        return out

    def stats(self) -> dict:
        s = Stats()
        check(lib().ssn_query(self._h, ctypes.byref(s)), "query")
        return s.as_dict()

    def device_logits_ptr(self) -> int:
        p = ctypes.c_void_p()
        check(lib().ssn_device_logits(self._h, ctypes.byref(p)), "device_logits")
        return p.value


def op_conv_bf16(x, n, h, w, cin, wgt, cout_max, cin_max, k, stride, pad, cout, scale=None,
                 shift=None, res=None, act=0, out_f32=0, y=None, stream=None):
    check(lib().ssn_op_conv_bf16(_ptr(x), n, h, w, cin, _ptr(wgt), cout_max, cin_max, k, stride,
                                 pad, cout, _ptr(scale), _ptr(shift), _ptr(res), act, out_f32,
                                 _ptr(y), _ptr(stream)), "op_conv_bf16")


def op_dw_bf16(x, n, h, w, c, wgt, c_max, k_max, k, stride, scale=None, shift=None, act=0,
               y=None, stream=None):
    """Depthwise bf16 operator (weights tap-major [k_max][k_max][c_max])."""
    check(lib().ssn_op_dw_bf16(_ptr(x), n, h, w, c, _ptr(wgt), c_max, k_max, k, stride,
                               _ptr(scale), _ptr(shift), act, _ptr(y), _ptr(stream)),
          "op_dw_bf16")


def op_conv_f32(x, n, h, w, cin, wgt, cout_max, cin_max, k_max, k, stride, pad, cout,
                depthwise=0, scale=None, shift=None, res=None, act=0, y=None, stream=None):
    check(lib().ssn_op_conv_f32(_ptr(x), n, h, w, cin, _ptr(wgt), cout_max, cin_max, k_max, k,
                                stride, pad, cout, depthwise, _ptr(scale), _ptr(shift), _ptr(res),
                                act, _ptr(y), _ptr(stream)), "op_conv_f32")
