"""oracle.direct -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

ctypes front-end of ``oracle/direct_conv.c``: the float64 direct N-D
cross-correlation of PAPER.md Eq. (2) (lines 137-141) with b = 0, f = id,
symmetric zero padding (readings #1-#3).  Also a pure-Python loop
version (`direct_conv_py`) used only for tiny brute-force pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "direct_conv.c"
_LIB = _HERE / "liboracle.so"
_lib = None


def build(force: bool = False) -> Path:
    """Compile liboracle.so with gcc (plain C, OpenMP)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(".so.tmp%d" % os.getpid())
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared",
                               str(_SRC), "-o", str(tmp)])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(_LIB))
        i64p = ctypes.POINTER(ctypes.c_int64)
        fp = ctypes.POINTER(ctypes.c_float)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_direct_conv_f64.argtypes = [ctypes.c_int, i64p, i64p, i64p, ctypes.c_int64,
                                               ctypes.c_int64, ctypes.c_int64, fp, fp, dp]
        lib.oracle_direct_conv_at.argtypes = [ctypes.c_int, i64p, i64p, i64p, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int64, fp, fp,
                                              ctypes.c_int64, i64p, dp]
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def _i64(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def out_dims(in_dims, r_dims, pad):
    """out_n = in_n + 2 P_n - r_n + 1 (SPEC.md:279 with symmetric padding)."""
    return tuple(int(i) + 2 * int(p) - int(r) + 1 for i, r, p in zip(in_dims, r_dims, pad))


def _prep(x, g, pad):
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    g = np.ascontiguousarray(np.asarray(g, dtype=np.float32))
    N = x.ndim - 2
    assert g.ndim == N + 2 and g.shape[1] == x.shape[1], "x [B][C][...], g [K][C][...]"
    if np.isscalar(pad):
        pad = (int(pad),) * N
    return x, g, N, tuple(int(p) for p in pad)


def direct_conv_f64(x, g, pad=0) -> np.ndarray:
    """Full y[b,k,o] in float64 (Eq. 2).  x: [B][C][in...], g: [K][C][r...]."""
    x, g, N, pad = _prep(x, g, pad)
    B, C = x.shape[:2]
    K = g.shape[0]
    od = out_dims(x.shape[2:], g.shape[2:], pad)
    if min(od) < 1:
        raise ValueError("kernel larger than padded input")
    y = np.empty((B, K) + od, dtype=np.float64)
    ind, indp = _i64(x.shape[2:])
    rd, rdp = _i64(g.shape[2:])
    pd, pdp = _i64(pad)
    st = _load().oracle_direct_conv_f64(
        N, indp, rdp, pdp, B, C, K,
        x.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        g.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        y.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if st:
        raise ValueError("oracle_direct_conv_f64 status %d" % st)
    return y


def direct_conv_at(x, g, pad, flat_idx) -> np.ndarray:
    """y.flat[flat_idx] computed one by one (for full-size sampled parity)."""
    x, g, N, pad = _prep(x, g, pad)
    B, C = x.shape[:2]
    K = g.shape[0]
    idx, idxp = _i64(flat_idx)
    vals = np.empty(idx.shape[0], dtype=np.float64)
    ind, indp = _i64(x.shape[2:])
    rd, rdp = _i64(g.shape[2:])
    pd, pdp = _i64(pad)
    st = _load().oracle_direct_conv_at(
        N, indp, rdp, pdp, B, C, K,
        x.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        g.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        idx.shape[0], idxp, vals.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if st:
        raise ValueError("oracle_direct_conv_at status %d" % st)
    return vals


def direct_conv_py(x, g, pad=0):
    """Pure-Python loops (tiny inputs only).  Works on any number type that
    supports + and * (ints, Fractions, floats): the brute-force sum of Eq. (2)."""
    x = np.asarray(x, dtype=object)
    g = np.asarray(g, dtype=object)
    N = x.ndim - 2
    if np.isscalar(pad):
        pad = (pad,) * N
    B, C = x.shape[:2]
    K = g.shape[0]
    ins, rs = x.shape[2:], g.shape[2:]
    od = out_dims(ins, rs, pad)
    y = np.empty((B, K) + od, dtype=object)
    for b in range(B):
        for k in range(K):
            for o in np.ndindex(*od):
                acc = 0
                for c in range(C):
                    for p in np.ndindex(*rs):
                        i = tuple(o[n] + p[n] - pad[n] for n in range(N))
                        if all(0 <= i[n] < ins[n] for n in range(N)):
                            acc = acc + g[(k, c) + p] * x[(b, c) + i]
                y[(b, k) + o] = acc
    return y
