"""Analytic cost model of the N-D Winograd layer.

CPU-only report; no kernel is launched.  The transform matrices come from
the library's exact host synthesis (`wino_synthesize`, C ABI), so zero
entries are exact zeros.

Paper side -- multiplication counts (Sec. 3.2-3.3, 4.1; fused
multiply-adds count as one multiplication, additions are free):

  theoretical_speedup(S, G, N) = (S G / D)^N, D = S + G - 1
  direct_muls(M, K, S, G, N)   = M K S^N G^N        per output tile (S^N outputs)
  fast_muls(M, K, AT, BT, N)   = D^N M K            element-wise products (Eq. (5))
                               + M * cost(B^T over N axes)   data transform, once per channel
                               + K * cost(A^T over N axes)   inverse, once per kernel
      (the kernel transform is cached).  A 1-D matrix X (rows x D) applied
      along axis n of the progressively transformed tile costs
      lines(n) * (rows * D dense | nnz(X) nonzero), lines(n) = prod of the other
      axes' current extents (axes before n already have `rows` entries).
  speedup_curve(...)           = direct / fast for K = M  (Figure 1)
  arithmetic_intensity(T, M, K, fused): 2 D^N M / 2 D^N M = 1
      unfused; 2 T K / (T + K) for the per-point matrix products of Eq. (5).

Paper slips reproduced as stated (reading #13): the sparse F(2, 3)
count is 18 by nonzero counting where P:178 prints 19 (and 4M^2 + 14M where
P:180 prints 4M^2 + 15M).

Device side -- the four-stage B200 pipeline of DESIGN.md Sec. 8: algorithmic
bytes and flops per stage (x, V, U, M, y each moved once) and the roofline
time at given peaks (HBM GB/s; 3xTF32 fp32-equivalent TFLOP/s for the GEMM).
"""
from __future__ import annotations

import argparse
import math
from fractions import Fraction
from typing import Dict, List, Sequence

from .wino import wino_synthesize


# ------------------------------------------------------------------ paper
def theoretical_speedup(S: int, G: int, N: int) -> Fraction:
    """(S G / D)^N exactly."""
    if S < 1 or G < 1 or N < 1:
        raise ValueError("S, G, N >= 1")
    return Fraction(S * G, S + G - 1) ** N


def theoretical_speedup_axes(S: Sequence[int], G: Sequence[int]) -> Fraction:
    """prod_n S_n G_n / D_n for per-axis transforms (Eq. (4) applies one
    F(S_n, G_n) per axis; the N-D count factorises over the axes)."""
    out = Fraction(1)
    for s_, g_ in zip(S, G):
        out *= theoretical_speedup(s_, g_, 1)
    return out


def direct_muls(M: int, K: int, S: int, G: int, N: int) -> int:
    """Sliding-window multiplications for one S^N output tile, all M x K pairs."""
    return M * K * S ** N * G ** N


def _entries(X) -> List[List[Fraction]]:
    return [[Fraction(v) for v in row] for row in X]


def nmode_cost(X, N: int, counting: str = "dense") -> int:
    """Multiplications to apply X (rows x D) along every axis 1..N of a D^N
    tensor, in axis order, each axis on the already-transformed tensor."""
    if counting not in ("dense", "nonzero"):
        raise ValueError("counting is 'dense' or 'nonzero'")
    X = _entries(X)
    rows, D = len(X), len(X[0])
    per_line = rows * D if counting == "dense" else sum(1 for r in X for v in r if v != 0)
    total = 0
    for n in range(N):
        lines = rows ** n * D ** (N - 1 - n)     # axes < n already have `rows` entries
        total += lines * per_line
    return total


def fast_muls(M: int, K: int, AT, BT, N: int, counting: str = "dense") -> int:
    """Multiplications of the fast algorithm for one output tile (kernel
    transform cached): D^N M K + M cost(B^T) + K cost(A^T)."""
    D = len(_entries(BT))
    return D ** N * M * K + M * nmode_cost(BT, N, counting) + K * nmode_cost(AT, N, counting)


def transforms(m: int, r: int, points: str = None) -> Dict[str, list]:
    """Exact A^T (m x alpha), G (alpha x r), B^T (alpha x alpha) from the
    library's synthesis (the same matrices the plans use)."""
    d = wino_synthesize(m, r, points)
    return {"AT": _entries(d["AT"]), "G": _entries(d["G"]), "BT": _entries(d["BT"]), "points": d["points"]}


def speedup_curve(m: int, r: int, N: int, Ms: Sequence[int], counting: str = "dense", points: str = None):
    """[(M, direct / fast)] with K = M (Figure 1's axes), plus the ceiling."""
    t = transforms(m, r, points)
    out = []
    for M in Ms:
        out.append((M, Fraction(direct_muls(M, M, m, r, N), fast_muls(M, M, t["AT"], t["BT"], N, counting))))
    return out


def arithmetic_intensity(T: int, M: int, K: int, fused: bool) -> Fraction:
    """Computations / memory accesses of the element-wise stage."""
    if min(T, M, K) < 1:
        raise ValueError("T, M, K >= 1")
    return Fraction(2 * T * K, T + K) if fused else Fraction(1)


# ------------------------------------------------------------------ device
def stage_model(N: int, dims: Sequence[int], m, r, C: int, K: int, B: int,
                pad: Sequence[int] = None, hbm_gbs: float = None, tf32_tflops: float = None,
                fold: int = 0, fold_mode: int = 0) -> Dict[str, dict]:
    """Algorithmic bytes / flops of the four stages of one forward (fp32,
    every tensor moved once) and, if peaks are given, the
    roofline time in ms of each stage (the GEMM at the 3xTF32 rate =
    tf32_tflops / 3 fp32-equivalent).  m and r may be per-axis sequences
    (F(m_1 x .. x m_N, r_1 x .. x r_N), Eq. (4)).

    fold = F > 0 (a5, single (m, r)): the GEMM writes W, (m/alpha)^F of M's
    size, and a4 reads W.  fold_mode 2 (the filter-side fold) reads U' = m^F
    x U and executes m^F x the multiply-adds (zero coefficients included);
    fold_mode 1 (epilogue fold) keeps U and the flops.  fold_mode 3 (the
    direct-axis fold, F = 1): a2 writes and the GEMM reads Z -- the input
    transformed along the outer axes only, (m t + alpha - m) raw columns per
    row of t tiles of the last axis -- instead of V, U' = m x U as in mode 2,
    and the GEMM executes the last axis directly: m r / alpha x the
    multiply-adds."""
    pad = tuple(pad) if pad is not None else (0,) * N
    mv = tuple(m) if isinstance(m, (list, tuple)) else (m,) * N
    rv = tuple(r) if isinstance(r, (list, tuple)) else (r,) * N
    out = [d + 2 * p - rn + 1 for d, p, rn in zip(dims, pad, rv)]
    T = B * math.prod(-(-o // mn) for o, mn in zip(out, mv))
    P = math.prod(mn + rn - 1 for mn, rn in zip(mv, rv))
    xb = 4 * B * C * math.prod(dims)
    yb = 4 * B * K * math.prod(out)
    # U counted once in fp32 (the compulsory filter bytes; the 3xTF32 GEMM
    # streams its hi/lo halves, i.e. 2x this, from L2)
    Vb, Mb, Ub = 4 * P * C * T, 4 * P * K * T, 4 * P * C * K
    gflops = 2 * P * T * C * K
    if fold:
        a, mm = mv[0] + rv[0] - 1, mv[0]
        Mb = Mb * mm ** fold // a ** fold            # W
        if fold_mode == 2:
            Ub *= mm ** fold                          # U'
            gflops *= mm ** fold
        elif fold_mode == 3:
            if fold != 1:
                raise ValueError("the direct-axis fold is F = 1")
            tl = -(-out[-1] // mm)                    # tiles along the last axis
            Vb = 4 * (P // a) * C * (T // tl) * (mm * tl + a - mm)      # Z
            Ub *= mm
            gflops = gflops * mm * rv[0] // a
    st = {
        "filter_xform": {"bytes": 4 * K * C * math.prod(rv) + Ub, "flops": 0},
        "input_xform": {"bytes": xb + Vb, "flops": 0},
        "gemm": {"bytes": Vb + Ub + Mb, "flops": gflops},
        "output_xform": {"bytes": Mb + yb, "flops": 0},
    }
    if hbm_gbs:
        for s in st.values():
            t_mem = s["bytes"] / (hbm_gbs * 1e9)
            t_tc = s["flops"] / (tf32_tflops / 3 * 1e12) if (tf32_tflops and s["flops"]) else 0.0
            s["roofline_ms"] = 1e3 * max(t_mem, t_tc)
            s["bound"] = "tensor" if t_tc > t_mem else "hbm"
    st["direct_flops"] = 2 * B * K * C * math.prod(out) * math.prod(rv)
    st["tiles"] = T
    return st


# ------------------------------------------------------------------ CLI
def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="Analytic cost report (CSV) of F(m^N, r^N)")
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--r", type=int, default=3)
    ap.add_argument("--N", type=int, default=3)
    ap.add_argument("--points", default=None)
    ap.add_argument("--Ms", default="1,2,5,10,20,50,100,200,500,1000")
    a = ap.parse_args(argv)
    t = transforms(a.m, a.r, a.points)
    ceil = theoretical_speedup(a.m, a.r, a.N)
    print("# F(%d^%d,%d^%d) points %s; ceiling (SG/D)^N = %.4f" % (a.m, a.N, a.r, a.N, ",".join(t["points"]),
                                                                float(ceil)))
    print("M,K,direct_muls,fast_muls_dense,fast_muls_sparse,ratio_dense,ratio_sparse,ceiling")
    for M in [int(v) for v in a.Ms.split(",")]:
        dm = direct_muls(M, M, a.m, a.r, a.N)
        fd = fast_muls(M, M, t["AT"], t["BT"], a.N, "dense")
        fs = fast_muls(M, M, t["AT"], t["BT"], a.N, "nonzero")
        print("%d,%d,%d,%d,%d,%.4f,%.4f,%.4f" % (M, M, dm, fd, fs, dm / fd, dm / fs, float(ceil)))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
