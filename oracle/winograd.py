"""oracle.winograd -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The N-dimensional fast convolution of PAPER.md Sec. 3.2-3.3 and 4.1, step by
step, over exact ``Fraction`` (object arrays) or float64:

1. tiling into overlapping D^N tiles stepping by S (
   DESIGN.md readings #2, #10: symmetric zero padding P, out = in + 2P - G + 1,
   ceil(out/S) tiles per axis, tile t reads input [tS - P, tS - P + D)
   zero-filled, outputs past `out` discarded);
2. kernel transform  G x_{n=1}^N C_n   (Eq. (4)),
   data transform    D x_{n=1}^N B_n  (one F(S_n, G_n) per axis allowed),
   each a chain of n-mode products (Eq. (3));
3. per transform point i: S_hat^(i) = D_hat^(i) x G_hat^(i) with D_hat T x M
   (tiles-by-channels) and G_hat M x K (Eq. (5)) -- the
   element-wise product fused with the channel reduction;
4. inverse transform  x_{n=1}^N A_n  and stitching.

Matrices use the paper's orientation: A (S x D), B (D x D), C (D x G).
No blocking, fusion or reordering beyond what Eq. (3)-(5) state.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


def as_array(Mx, exact: bool):
    if exact:
        return np.array([[Fraction(v) for v in row] for row in Mx], dtype=object)
    return np.array([[float(v) for v in row] for row in Mx], dtype=np.float64)


def nmode_product(X: np.ndarray, U: np.ndarray, n: int) -> np.ndarray:
    """(X x_n U)_{i1..j..iN} = sum_{i_n} x_{i1..i_n..iN} u_{j,i_n}  (Eq. (3))."""
    Y = np.tensordot(U, X, axes=([1], [n]))     # new axis j first
    return np.moveaxis(Y, 0, n)


def multi_mode_product(X: np.ndarray, U: np.ndarray, axes) -> np.ndarray:
    """X x_{n} U over the listed axes, left to right."""
    for ax in axes:
        X = nmode_product(X, U, ax)
    return X


def _per_axis(v, N):
    """An int or a length-N sequence -> tuple of N ints."""
    return tuple(int(a) for a in v) if isinstance(v, (list, tuple)) else (int(v),) * N


def tile_geometry(in_dims, r, m, pad):
    """out dims, tiles per axis, T per sample (readings #2, #10); r and m may
    be per-axis sequences (Eq. (4) indexes the transforms by axis n)."""
    N = len(in_dims)
    r, m = _per_axis(r, N), _per_axis(m, N)
    out = tuple(int(i) + 2 * int(p) - rn + 1 for i, p, rn in zip(in_dims, pad, r))
    tiles = tuple(math.ceil(o / mn) for o, mn in zip(out, m))
    return out, tiles


def extract_tiles(x: np.ndarray, m, alpha, pad, zero):
    """x [B][C][in...] -> tiles [B][C][t_1..t_N][alpha_1..alpha_N], zero-filled:
    tile t, window position w reads x at t_n m_n - P_n + w_n (zero outside
    [0, in_n)), readings #2, #10.  Written as: zero-extend x by P_n before and
    as far as the last window reaches after, then for every window position w
    take the strided slice w_n, w_n + m_n, ... along each axis."""
    N = x.ndim - 2
    m, alpha = _per_axis(m, N), _per_axis(alpha, N)
    r = tuple(a - mn + 1 for a, mn in zip(alpha, m))
    out, tiles = tile_geometry(x.shape[2:], r, m, pad)
    span = tuple(tiles[n] * m[n] + alpha[n] - m[n] for n in range(N))     # padded extent the tiles read
    xp = np.empty(x.shape[:2] + span, dtype=x.dtype)
    xp[...] = zero
    src, dst = [], []
    for n in range(N):
        lo, hi = pad[n], min(span[n], pad[n] + x.shape[2 + n])             # x index i lands at i + P_n
        dst.append(slice(lo, hi))
        src.append(slice(0, hi - lo))
    xp[(slice(None), slice(None)) + tuple(dst)] = x[(slice(None), slice(None)) + tuple(src)]
    res = np.empty(x.shape[:2] + tiles + alpha, dtype=x.dtype)
    for w in np.ndindex(*alpha):
        sl = tuple(slice(w[n], w[n] + m[n] * tiles[n], m[n]) for n in range(N))
        res[(slice(None), slice(None)) + tuple(slice(None) for _ in range(N)) + w] = xp[(slice(None), slice(None)) + sl]
    return res, out, tiles


def winograd_nd(x, g, pad, A, B, C, exact: bool = False):
    """Full N-D Winograd layer.  Returns (y, stages) where stages holds
    U [P][M][K] (G_hat^(i)), V [P][T][M] (D_hat^(i)), Shat [P][T][K]
    (S_hat^(i)), P = prod_n D_n, with i row-major over the transform-domain
    coordinates and t row-major over (b, t_1..t_N).

    A, B, C are one matrix each (the same F(S, G) on every axis) or lists of
    N matrices A_n (S_n x D_n), B_n (D_n x D_n), C_n (D_n x G_n): Eq. (4)
    applies x_n with the n-th transform."""
    if exact:
        x = np.asarray(x, dtype=object)
        g = np.asarray(g, dtype=object)
        zero = Fraction(0)
    else:
        x = np.asarray(x, dtype=np.float64)
        g = np.asarray(g, dtype=np.float64)
        zero = 0.0
    N = x.ndim - 2

    def axes_list(Mx):
        # a single matrix (list of rows of scalars) or a list of N matrices
        if isinstance(Mx, (list, tuple)) and len(Mx) == N and np.ndim(np.asarray(Mx[0], dtype=object)) == 2:
            return [as_array(Mi, exact) for Mi in Mx]
        return [as_array(Mx, exact)] * N

    As, Bs, Cs = axes_list(A), axes_list(B), axes_list(C)
    S = tuple(a.shape[0] for a in As)
    D = tuple(a.shape[1] for a in As)
    Gk = tuple(c.shape[1] for c in Cs)
    if np.isscalar(pad):
        pad = (int(pad),) * N
    Bn, M = x.shape[:2]
    K = g.shape[0]
    assert g.shape[2:] == Gk

    # (2) kernel transform: G x_{n=1}^N C_n  -> [K][M][D_1..D_N]
    Ug = g
    for n in range(N):
        Ug = nmode_product(Ug, Cs[n], 2 + n)
    # (1)+(2) tiles and data transform: D x_{n=1}^N B_n
    tiles, out, tgrid = extract_tiles(x, S, D, pad, zero)
    Vt = tiles
    for n in range(N):
        Vt = nmode_product(Vt, Bs[n], 2 + N + n)                   # [B][M][tiles][D..]
    T = Bn * int(np.prod(tgrid))
    P = int(np.prod(D))
    # i-major matrices of Eq. (5)
    Ghat = Ug.reshape(K, M, P).transpose(2, 1, 0)                     # [P][M][K]
    Dhat = np.moveaxis(Vt, 1, -1 - N)                                 # [B][tiles][M][D..]
    Dhat = Dhat.reshape(T, M, P).transpose(2, 0, 1)                   # [P][T][M]
    # (3) per transform point: S_hat^(i) = D_hat^(i) G_hat^(i)
    Shat = np.empty((P, T, K), dtype=Dhat.dtype)
    for i in range(P):
        Shat[i] = np.dot(Dhat[i], Ghat[i])
    # (4) inverse transform per (t, k) and stitch
    Yt = Shat.transpose(1, 2, 0).reshape((T, K) + D)
    for n in range(N):
        Yt = nmode_product(Yt, As[n], 2 + n)                          # [T][K][S..]
    Yt = Yt.reshape((Bn,) + tgrid + (K,) + S)
    # stitch: output o of tile t lands at t_n S_n + o_n; outputs past `out` are discarded
    order = [0, 1 + N] + [a for n in range(N) for a in (1 + n, 2 + N + n)]   # [B][K][t_1][S_1]..[t_N][S_N]
    full = Yt.transpose(order).reshape((Bn, K) + tuple(tgrid[n] * S[n] for n in range(N)))
    y = np.ascontiguousarray(full[(slice(None), slice(None)) + tuple(slice(0, o) for o in out)])
    return y, {"U": Ghat, "V": Dhat, "Shat": Shat, "out": out, "tiles": tgrid}


def winograd_2d_closed_form(d_tile, g_ker, A, B, C, exact: bool = False):
    """The 2-D special case S = A[(C G C^T) (.) (B D B^T)] A^T."""
    A_, B_, C_ = as_array(A, exact), as_array(B, exact), as_array(C, exact)
    dt = np.asarray(d_tile, dtype=object if exact else np.float64)
    gk = np.asarray(g_ker, dtype=object if exact else np.float64)
    return A_.dot((C_.dot(gk).dot(C_.T)) * (B_.dot(dt).dot(B_.T))).dot(A_.T)
