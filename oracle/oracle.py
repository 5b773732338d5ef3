"""ctypes wrapper of the CPU oracle (liboracle.so) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module (see oracle/ssn_oracle.c for what it restates and how parity is
pinned).  The product path never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_BIN = os.path.join(HERE, "_ref", "servesim_ref")
_L = None


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("depth_flags", ctypes.POINTER(ctypes.c_uint8)), ("n_depth", ctypes.c_uint32),
        ("expand_ratios", ctypes.POINTER(ctypes.c_double)), ("n_expand", ctypes.c_uint32),
        ("width_multipliers", ctypes.POINTER(ctypes.c_double)), ("n_width", ctypes.c_uint32),
        ("kernel_sizes", ctypes.POINTER(ctypes.c_uint32)), ("n_kernel", ctypes.c_uint32),
    ]


def build():
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)


def lib():
    global _L
    if _L is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        P, i32, u32, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64
        cp = ctypes.POINTER(_Cfg)
        L.oracle_create.restype = P
        L.oracle_create.argtypes = [i32, u64, i32, i32]
        L.oracle_destroy.argtypes = [P]
        L.oracle_stat_count.restype = ctypes.c_long
        L.oracle_stat_count.argtypes = [P, cp]
        L.oracle_forward.restype = i32
        L.oracle_forward.argtypes = [P, cp, u32, P, i32, i32, P, P, i32, P, P, P]
        L.oracle_last_error.restype = ctypes.c_char_p
        L.oracle_weight.restype = ctypes.c_float
        L.oracle_weight.argtypes = [P, i32, i32, i32, i32, i32]
        L.oracle_num_tensors.argtypes = [P]
        L.oracle_set_threads.argtypes = [i32]
        L.oracle_images.argtypes = [u64, u32, i32, i32, P]
        L.oracle_forward_tokens.restype = i32
        L.oracle_forward_tokens.argtypes = [P, cp, P, i32, i32, i32, P]
        L.oracle_tokens.argtypes = [u64, u32, i32, i32, P]
        L.oracle_conv_op.restype = i32
        L.oracle_conv_op.argtypes = [P, i32, i32, i32, i32, P, i32, i32, i32, i32, i32, i32,
                                     i32, i32, P, P, P, i32, P]
        _L = L
    return _L


def _cfg(cfg):
    d = (ctypes.c_uint8 * len(cfg.depth_flags))(*[1 if f else 0 for f in cfg.depth_flags])
    e = (ctypes.c_double * len(cfg.expand_ratios))(*cfg.expand_ratios)
    w = (ctypes.c_double * len(cfg.width_multipliers))(*cfg.width_multipliers)
    ks = list(getattr(cfg, "kernel_sizes", []) or [])
    k = (ctypes.c_uint32 * max(1, len(ks)))(*ks)
    s = _Cfg(ctypes.cast(d, ctypes.POINTER(ctypes.c_uint8)), len(d),
             ctypes.cast(e, ctypes.POINTER(ctypes.c_double)), len(e),
             ctypes.cast(w, ctypes.POINTER(ctypes.c_double)), len(w),
             ctypes.cast(k, ctypes.POINTER(ctypes.c_uint32)) if ks else None, len(ks))
    return s, (d, e, w, k)


def _p(a):
    return None if a is None else a.ctypes.data


class OracleNet:
    FLAG_BF16_STORAGE = 1
    FLAG_CALIBRATE = 2

    def __init__(self, family: int, seed: int = 0, classes: int = 1000, bf16_weights: bool = True):
        self.family, self.classes = family, classes
        self.h = lib().oracle_create(family, seed, classes, int(bf16_weights))
        if not self.h:
            raise ValueError(lib().oracle_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_destroy(self.h)
            self.h = None

    def stat_count(self, cfg) -> int:
        s, keep = _cfg(cfg)
        n = lib().oracle_stat_count(self.h, ctypes.byref(s))
        if n < 0:
            raise ValueError(lib().oracle_last_error().decode())
        return n

    def weight(self, tensor, co, ci, r, s):
        return lib().oracle_weight(self.h, tensor, co, ci, r, s)

    def forward(self, cfg, x_nchw, subnet_id=0, mean=None, var=None, bf16_storage=False):
        x = np.ascontiguousarray(x_nchw, dtype=np.float32)
        n, _, hw, _ = x.shape
        out = np.zeros((n, self.classes), dtype=np.float32)
        s, keep = _cfg(cfg)
        if mean is not None:
            mean = np.ascontiguousarray(mean, np.float32)
            var = np.ascontiguousarray(var, np.float32)
        rc = lib().oracle_forward(self.h, ctypes.byref(s), subnet_id, _p(x), n, hw, _p(mean),
                                  _p(var), self.FLAG_BF16_STORAGE if bf16_storage else 0,
                                  _p(out), None, None)
        if rc:
            raise ValueError(lib().oracle_last_error().decode())
        return out

    def forward_tokens(self, cfg, ids, bf16_storage=False, acc64=False):
        """BERT logits; acc64 accumulates the linears in double (a second,
        equally valid implementation of the same bf16-storage semantics: the
        spread between the two measures how implementation-sensitive the
        bf16-stored network is on these inputs)."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        n, seq = ids.shape
        out = np.zeros((n, self.classes), dtype=np.float32)
        s, keep = _cfg(cfg)
        flags = (1 if bf16_storage else 0) | (4 if acc64 else 0)
        rc = lib().oracle_forward_tokens(self.h, ctypes.byref(s), _p(ids), n, seq, flags,
                                         _p(out))
        if rc:
            raise ValueError(lib().oracle_last_error().decode())
        return out

    def calibrate(self, cfg, x_nchw):
        """SubnetNorm calibration: per-subnet (mu, var) from batch statistics."""
        x = np.ascontiguousarray(x_nchw, dtype=np.float32)
        n, _, hw, _ = x.shape
        cnt = self.stat_count(cfg)
        mean = np.zeros(cnt, np.float32)
        var = np.zeros(cnt, np.float32)
        s, keep = _cfg(cfg)
        rc = lib().oracle_forward(self.h, ctypes.byref(s), 0, _p(x), n, hw, None, None,
                                  self.FLAG_CALIBRATE, None, _p(mean), _p(var))
        if rc:
            raise ValueError(lib().oracle_last_error().decode())
        return mean, var


def images(seed: int, batch_ordinal: int, n: int, hw: int) -> np.ndarray:
    out = np.zeros((n, 3, hw, hw), np.float32)
    lib().oracle_images(seed, batch_ordinal, n, hw, out.ctypes.data)
    return out


def tokens(seed: int, batch_ordinal: int, n: int, seq: int) -> np.ndarray:
    out = np.zeros((n, seq), np.int32)
    lib().oracle_tokens(seed, batch_ordinal, n, seq, out.ctypes.data)
    return out


def conv_op(x_nhwc, wgt_oihw, cout_max, cin_max, k_max, k, stride, pad, cout, depthwise=False,
            scale=None, shift=None, res=None, act=0):
    x = np.ascontiguousarray(x_nhwc, np.float32)
    n, h, w, cin = x.shape
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    y = np.zeros((n, ho, wo, cout), np.float32)
    wgt = np.ascontiguousarray(wgt_oihw, np.float32)
    f = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)
    scale, shift, res = f(scale), f(shift), f(res)
    lib().oracle_conv_op(_p(x), n, h, w, cin, _p(wgt), cout_max, cin_max, k_max, k, stride, pad,
                         cout, int(depthwise), _p(scale), _p(shift), _p(res), act, _p(y))
    return y


def set_threads(n: int):
    lib().oracle_set_threads(n)


def ref_available() -> bool:
    return os.path.exists(REF_BIN)


def ref_decide(catalog: str, buckets: int, slacks):
    """Reference SlackFit decisions (policy.hpp:191) via oracle/_ref."""
    out = subprocess.run([REF_BIN, "decide", catalog, str(buckets)] + [str(s) for s in slacks],
                         check=True, capture_output=True, text=True).stdout
    res = []
    for line in out.strip().splitlines():
        parts = line.split()
        res.append(None if parts[1] == "drop" else (int(parts[1]), int(parts[2]), int(parts[3])))
    return res
