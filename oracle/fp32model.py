"""oracle.fp32model -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

A float32 model of the rounding the device arithmetic performs in the N-D
fast convolution of Eq. (3)-(5).  Its purpose is
the parity tolerance of the GPU tests wherever BASELINE.json states none
(arbitrary (m, r), per-axis transforms, the paper's 2-D nets; DESIGN.md
readings #15, #17): the bound is k x the error of this model on the same
seeded inputs, so it comes from the arithmetic, not from the device under
test.  PAPER.md:96 names numeric stability as the price of non-simple
transforms; this model makes that price computable per (m, r, N, points).

It is built only from ``oracle.toomcook`` (the exact-rational synthesis) and
``oracle.winograd`` (tiling and n-mode products), and follows
``oracle.winograd.winograd_nd`` step by step with the rounding of each step
made explicit (reading #7):

1. kernel transform U = g x_n C_n in float64 from the fp32 weights, rounded
   once to float32;
2. constants A_n, B_n rounded to nearest-even float32 from the exact
   rationals (``f32_rne``, no double rounding through float64);
3. data transform V = tiles x_n B_n in float32 (one float32 n-mode product
   per axis, numpy tensordot);
4. per-point product, one of
   * ``"f64"``:         float64 (no rounding: the model then equals
                        oracle.winograd's float64 result),
   * ``"fp32"``:        float32 matmul (numpy sgemm),
   * ``"fp32_seq"``:    float32, accumulated sequentially over channels,
   * ``"3xtf32_k8"``:   the tensor-core model: V = V_hi + V_lo, U = U_hi +
                        U_lo with hi = tf32_rna(x), lo = tf32_rna(x - hi);
                        per block of 8 channels the three products V_lo U_hi
                        + V_hi U_lo + V_hi U_hi are summed exactly (float64)
                        and added to a float32 accumulator with one
                        round-to-nearest-even,
   * ``"1xtf32_k8"``:   V_hi U_hi only (what a single TF32 product gives);
   * ``"3xf16_k16"``:   the kind::f16 scheme (gemm_f16.cu): V and U scaled by
                        powers of two to a largest magnitude <= 2^15 and split
                        into fp16 hi + lo (round to nearest even), three
                        products per block of 16 channels, fp32 accumulation;
5. inverse transform y = S_hat x_n A_n in float32.

The tensor core's internal K=8 summation precision and its TMEM accumulation
rounding are not documented (SURVEY.md Appendix B caveat); the k factor of
the tolerance covers that, and the summation order, which differs between
this model and the device.
"""
from __future__ import annotations

import math
from fractions import Fraction
from typing import Sequence

import numpy as np

from . import toomcook as tc
from .winograd import extract_tiles, nmode_product, tile_geometry


# ------------------------------------------------------------ rounding
def f32_rne(q) -> np.float32:
    """The float32 nearest to the exact rational q, ties to even."""
    q = Fraction(q)
    c = np.float32(float(q))                   # within one float32 ulp of q
    best = None
    for cand in (np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))):
        d = abs(Fraction(float(cand)) - q)
        key = (d, int(np.array(cand, dtype=np.float32).view(np.uint32)) & 1)   # ties -> even mantissa
        if best is None or key < best[0]:
            best = (key, cand)
    return np.float32(best[1])


def tf32_rna(a) -> np.ndarray:
    """Round float32 values to TF32 (10 explicit mantissa bits), ties away
    from zero -- cvt.rna.tf32.f32 (reading #7).  The result is a
    float32 with its low 13 mantissa bits zero."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    bits = a.view(np.uint32).astype(np.uint64)
    finite = np.isfinite(a)
    # sign-magnitude: adding half an ulp (bit 12) to the magnitude rounds half away
    out = np.where(finite, (bits + 0x1000) & ~np.uint64(0x1FFF), bits).astype(np.uint32)
    return out.view(np.float32).reshape(a.shape)


def split_tf32(a):
    """(hi, lo) with hi = tf32_rna(a), lo = tf32_rna(a - hi) (float32)."""
    a = np.asarray(a, dtype=np.float32)
    hi = tf32_rna(a)
    lo = tf32_rna((a - hi).astype(np.float32))
    return hi, lo


# ------------------------------------------------------------ points
def default_points(alpha: int) -> list:
    """DESIGN.md reading #5: alpha = 4: {0, 1, -1, inf}; alpha = 6:
    {0, 3/2, -3/2, 2/3, -2/3, inf}; otherwise SPEC.md:138's order 0, 1, -1,
    2, -2, 1/2, -1/2, 3, -3, ... with the last point at infinity (alpha = 1:
    the single point 0, F(1,1) = identity)."""
    if alpha == 1:
        return [Fraction(0)]
    if alpha == 4:
        return tc.parse_points("0,1,-1,inf")
    if alpha == 6:
        return tc.parse_points("0,3/2,-3/2,2/3,-2/3,inf")
    seq = [Fraction(0), Fraction(1), Fraction(-1)]
    k = 2
    while len(seq) < alpha - 1:
        seq += [Fraction(k), Fraction(-k), Fraction(1, k), Fraction(-1, k)]
        k += 1
    return seq[:alpha - 1] + [tc.INF]


def transforms(m: int, r: int, points=None):
    """(A, B, C) exact for F(m, r) from oracle.toomcook (default points if None)."""
    pts = default_points(m + r - 1) if points is None else points
    return tc.synthesize(m, r, pts)


# ------------------------------------------------------------ the product
def gemm_model(Vp: np.ndarray, Up: np.ndarray, mode: str) -> np.ndarray:
    """S_hat = V U for one transform point (Eq. (5)): V [T][M] float32,
    U [M][K] float32, in the rounding `mode` (module docstring, step 4)."""
    if mode == "f64":
        return Vp.astype(np.float64) @ Up.astype(np.float64)
    if mode == "fp32":
        return (Vp.astype(np.float32) @ Up.astype(np.float32)).astype(np.float32)
    T, M = Vp.shape
    K = Up.shape[1]
    if mode == "fp32_seq":
        acc = np.zeros((T, K), dtype=np.float32)
        for c in range(M):
            acc = (acc + np.outer(Vp[:, c], Up[c]).astype(np.float32)).astype(np.float32)
        return acc
    if mode == "3xf16_k16":
        # the kind::f16 scheme: V and U scaled by powers of two so that their
        # largest magnitude is <= 2^15, each split into fp16 hi + lo (round to
        # nearest even); per block of 16 channels lo*hi + hi*lo + hi*hi summed
        # exactly, one fp32 rounding into the accumulator; result scaled back
        def split16(a):
            a = np.asarray(a, dtype=np.float32)
            m = float(np.abs(a).max()) if a.size else 0.0
            s = 0 if m == 0.0 else int(np.floor(np.log2(m))) + 1 - 15
            sc = np.float32(2.0 ** -s)
            a2 = (a * sc).astype(np.float32)
            hi = a2.astype(np.float16)
            lo = (a2 - hi.astype(np.float32)).astype(np.float16)
            return hi.astype(np.float64), lo.astype(np.float64), s
        vh, vl, sv = split16(Vp)
        uh, ul, su = split16(Up)
        acc = np.zeros((T, K), dtype=np.float32)
        for c0 in range(0, M, 16):
            b = slice(c0, min(M, c0 + 16))
            blk = vl[:, b] @ uh[b] + vh[:, b] @ ul[b] + vh[:, b] @ uh[b]
            acc = (acc.astype(np.float64) + blk).astype(np.float32)
        return (acc.astype(np.float64) * 2.0 ** (sv + su)).astype(np.float32)
    if mode in ("3xtf32_k8", "1xtf32_k8"):
        vh, vl = split_tf32(Vp)
        uh, ul = split_tf32(Up)
        vh, vl, uh, ul = (a.astype(np.float64) for a in (vh, vl, uh, ul))
        acc = np.zeros((T, K), dtype=np.float32)
        for c0 in range(0, M, 8):
            b = slice(c0, min(M, c0 + 8))
            if mode == "3xtf32_k8":
                blk = vl[:, b] @ uh[b] + vh[:, b] @ ul[b] + vh[:, b] @ uh[b]
            else:
                blk = vh[:, b] @ uh[b]
            acc = (acc.astype(np.float64) + blk).astype(np.float32)
        return acc
    raise ValueError("unknown mode %r" % mode)


def winograd_model(x, g, pad, m, r, points=None, mode: str = "3xtf32_k8"):
    """The layer y = Eq. (2) (b = 0, f = id) computed by Eq. (4)-(5) with the
    device's rounding (module docstring).  x [B][M][in...] and g [K][M][r...]
    hold float32 values; m, r: an int or per-axis sequences (Eq. (4));
    points: None (defaults) or one list for every axis.  Returns y as float32
    (float64 in mode "f64")."""
    x = np.asarray(x, dtype=np.float32)
    g = np.asarray(g, dtype=np.float64)
    N = x.ndim - 2
    ms = tuple(m) if isinstance(m, (list, tuple)) else (m,) * N
    rs = tuple(r) if isinstance(r, (list, tuple)) else (r,) * N
    pads = (int(pad),) * N if np.isscalar(pad) else tuple(int(p) for p in pad)
    mats = [transforms(ms[n], rs[n], points) for n in range(N)]
    exact64 = mode == "f64"
    ft = np.float64 if exact64 else np.float32
    As = [np.array([[float(v) if exact64 else f32_rne(v) for v in row] for row in A_], dtype=ft) for A_, _, _ in mats]
    Bs = [np.array([[float(v) if exact64 else f32_rne(v) for v in row] for row in B_], dtype=ft) for _, B_, _ in mats]
    Cs = [np.array([[float(v) for v in row] for row in C_], dtype=np.float64) for _, _, C_ in mats]
    S = tuple(a.shape[0] for a in As)
    D = tuple(a.shape[1] for a in As)
    Bn, M = x.shape[:2]
    K = g.shape[0]
    # 1. kernel transform in float64, one rounding to float32
    Ug = g
    for n in range(N):
        Ug = nmode_product(Ug, Cs[n], 2 + n)
    Ug = Ug.astype(ft)
    # 3. tiles and data transform in float32
    tiles, out, tgrid = extract_tiles(x.astype(ft), S, D, pads, ft(0))
    Vt = tiles
    for n in range(N):
        Vt = nmode_product(Vt, Bs[n], 2 + N + n).astype(ft)
    T = Bn * int(np.prod(tgrid))
    P = int(np.prod(D))
    Ghat = Ug.reshape(K, M, P).transpose(2, 1, 0)
    Dhat = np.moveaxis(Vt, 1, -1 - N).reshape(T, M, P).transpose(2, 0, 1)
    # 4. per-point products
    Shat = np.empty((P, T, K), dtype=ft)
    for i in range(P):
        Shat[i] = gemm_model(np.ascontiguousarray(Dhat[i]), np.ascontiguousarray(Ghat[i]), mode)
    # 5. inverse transform in float32 and stitching
    Yt = Shat.transpose(1, 2, 0).reshape((T, K) + D)
    for n in range(N):
        Yt = nmode_product(Yt, As[n], 2 + n).astype(ft)
    Yt = Yt.reshape((Bn,) + tgrid + (K,) + S)
    order = [0, 1 + N] + [a for n in range(N) for a in (1 + n, 2 + N + n)]
    full = Yt.transpose(order).reshape((Bn, K) + tuple(tgrid[n] * S[n] for n in range(N)))
    y = np.ascontiguousarray(full[(slice(None), slice(None)) + tuple(slice(0, o) for o in out)])
    return y


# ------------------------------------------------------------ tolerances
def errors(y, ref):
    """(relL2, max-abs / max|ref|) in float64."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = y - ref
    return float(np.linalg.norm(d) / np.linalg.norm(ref)), float(np.abs(d).max() / np.abs(ref).max())


K_REL, K_MAX = 4.0, 8.0


def model_tolerance(x, g, pad, m, r, ref, points=None, mode="3xtf32_k8"):
    """Parity bound for a GPU result on these inputs: (K_REL x the model's
    relL2, K_MAX x its max-abs / max|y|) against the float64 reference `ref`
    (reading #15).  Returns (tol_rel, tol_max, model_rel, model_max)."""
    y = winograd_model(x, g, pad, m, r, points, mode)
    rel, mx = errors(y, ref)
    return K_REL * rel, K_MAX * mx, rel, mx
