"""LR-CNN oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 CPU implementation of what the
row-centric training hot path computes (arXiv 2401.11471, PAPER.md).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The oracle
shares no code, header, table or helper with the CUDA product path in
``paper_2401_11471_b200/`` and never imports it.

Modules:
  column      -- layer-by-layer (column) FP/BP/SGD, Eqs. (1)-(2), Alg. 1 with N=1
  enumerate   -- brute-force row-dependency enumerator (set based)
  rowcentric  -- slow CPU row-centric executor (2PS, OverL, segments, rank sim.)
  memmodel    -- Eq. (3), (6)-(8), tau/iota FLOP formulas

Parity status: every function is pinned by tests/test_oracle_*.py; see
DESIGN.md "Oracle pins" for the list (no function is "parity unpinned").
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_ops.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# Portable flags: the .so is built on the dev host and may run on the GPU
# box's host CPU, so no -march=native.
CFLAGS = ["-O3", "-fopenmp", "-shared", "-fPIC", "-std=c11"]


def build(force=False):
    """Compile oracle_ops.c -> liboracle.so (gcc).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", _LIB, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        lp = ctypes.POINTER(ctypes.c_long)
        i = ctypes.c_int
        L.oracle_out_dim.argtypes = [i, i, i, i, i]
        L.oracle_out_dim.restype = i
        L.oracle_conv2d_fwd.argtypes = [i, i, i, i, dp, i, i, i, i, i, i, i, dp, dp, dp]
        L.oracle_conv2d_bwd_data.argtypes = [i, i, i, i, i, i, i, i, i, i, i, dp, dp, dp]
        L.oracle_conv2d_bwd_weight.argtypes = [i, i, i, i, dp, i, i, i, i, i, i, i, dp, dp, dp]
        L.oracle_maxpool_fwd.argtypes = [i, i, i, i, dp, i, i, i, i, i, i, dp, lp]
        L.oracle_maxpool_bwd.argtypes = [i, i, i, i, i, i, lp, dp, dp]
        for f in ("oracle_conv2d_fwd", "oracle_conv2d_bwd_data", "oracle_conv2d_bwd_weight",
                  "oracle_maxpool_fwd", "oracle_maxpool_bwd"):
            getattr(L, f).restype = None
        _lib = L
    return _lib


def set_threads(n):
    """Number of OpenMP threads the oracle uses (cpu_baseline reports it)."""
    os.environ["OMP_NUM_THREADS"] = str(int(n))
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def out_dim(h, pad_a, pad_b, k, s):
    """floor((h + pad_a + pad_b - k)/s) + 1  (PAPER.md:232 printed law is garbled)."""
    return lib().oracle_out_dim(h, pad_a, pad_b, k, s)


def conv2d_fwd(x, w, bias, s, pads):
    """Eq. (1): z = Conv(x, w) + bias.  x [B,Ci,H,W], w [Co,Ci,k,k], pads=(top,bottom,left,right)."""
    x = _c64(x)
    w = _c64(w)
    B, Ci, H, W = x.shape
    Co, Ci2, k, k2 = w.shape
    assert Ci == Ci2 and k == k2
    pt, pb, pl, pr = pads
    Ho, Wo = out_dim(H, pt, pb, k, s), out_dim(W, pl, pr, k, s)
    if Ho < 1 or Wo < 1:
        raise ValueError("kernel-exceeds-input")
    y = np.empty((B, Co, Ho, Wo))
    b = None if bias is None else _c64(bias)
    lib().oracle_conv2d_fwd(B, Ci, H, W, _dp(x), Co, k, s, pt, pb, pl, pr, _dp(w),
                            None if b is None else _dp(b), _dp(y))
    return y


def conv2d_bwd_data(w, dy, in_hw, s, pads):
    """Adjoint of conv2d_fwd w.r.t. its input (delta^{l-1} = Get_error(delta^l, theta^l), Alg. 1 l.17)."""
    w = _c64(w)
    dy = _c64(dy)
    B, Co, Ho, Wo = dy.shape
    Co2, Ci, k, _ = w.shape
    assert Co == Co2
    H, W = in_hw
    pt, pb, pl, pr = pads
    assert out_dim(H, pt, pb, k, s) == Ho and out_dim(W, pl, pr, k, s) == Wo
    dx = np.empty((B, Ci, H, W))
    lib().oracle_conv2d_bwd_data(B, Ci, H, W, Co, k, s, pt, pb, pl, pr, _dp(w), _dp(dy), _dp(dx))
    return dx


def conv2d_bwd_weight(x, dy, k, s, pads, with_bias=True):
    """Eq. (2): g = Gradient(delta, z^{l-1}); returns (dw [Co,Ci,k,k], db [Co] or None)."""
    x = _c64(x)
    dy = _c64(dy)
    B, Ci, H, W = x.shape
    B2, Co, Ho, Wo = dy.shape
    assert B == B2
    pt, pb, pl, pr = pads
    assert out_dim(H, pt, pb, k, s) == Ho and out_dim(W, pl, pr, k, s) == Wo
    dw = np.empty((Co, Ci, k, k))
    db = np.empty(Co) if with_bias else None
    lib().oracle_conv2d_bwd_weight(B, Ci, H, W, _dp(x), Co, k, s, pt, pb, pl, pr, _dp(dy), _dp(dw),
                                   None if db is None else _dp(db))
    return dw, db


def maxpool_fwd(x, k, s, pads):
    """Max pooling; ties -> lowest flat index; pads never win."""
    x = _c64(x)
    B, C, H, W = x.shape
    pt, pb, pl, pr = pads
    Ho, Wo = out_dim(H, pt, pb, k, s), out_dim(W, pl, pr, k, s)
    if Ho < 1 or Wo < 1:
        raise ValueError("kernel-exceeds-input")
    y = np.empty((B, C, Ho, Wo))
    am = np.empty((B, C, Ho, Wo), dtype=np.int64)
    lib().oracle_maxpool_fwd(B, C, H, W, _dp(x), k, s, pt, pb, pl, pr, _dp(y),
                             am.ctypes.data_as(ctypes.POINTER(ctypes.c_long)))
    return y, am


def maxpool_bwd(argmax, dy, in_hw):
    """Route each delta to its argmax (adjoint of maxpool_fwd)."""
    dy = _c64(dy)
    am = np.ascontiguousarray(argmax, dtype=np.int64)
    B, C, Ho, Wo = dy.shape
    H, W = in_hw
    dx = np.empty((B, C, H, W))
    lib().oracle_maxpool_bwd(B, C, H, W, Ho, Wo, am.ctypes.data_as(ctypes.POINTER(ctypes.c_long)),
                             _dp(dy), _dp(dx))
    return dx
