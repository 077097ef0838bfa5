"""Pins for oracle.winograd (the N-D algorithm of Eq. (3)-(5), step by step).

Pinned against: brute-force direct correlation in exact rationals (two
different definitions must agree exactly, "S = ..."); the 2-D
closed form A(CGC^T (.) BDB^T)A^T; the tile-count example
of SPEC.md:208; and the C float64 direct oracle at small float shapes.
"""
import random
from fractions import Fraction as F

import numpy as np
import pytest

from oracle import direct, toomcook as tc, winograd as wg


def _rand_frac(rng, shape):
    flat = [F(rng.randint(-9, 9), rng.randint(1, 4)) for _ in range(int(np.prod(shape)))]
    return np.array(flat, dtype=object).reshape(shape)


CASES = [
    # N, S(m), G(r), pad, spatial, B, C, K
    (1, 2, 3, 0, (7,), 1, 2, 2),      # length 7, D=4, S=2 -> 3 tiles (partial)
    (1, 4, 3, 1, (9,), 2, 2, 2),
    (1, 3, 2, 2, (5,), 1, 2, 2),
    (2, 2, 3, 1, (5, 6), 1, 2, 2),
    (2, 4, 3, 1, (6, 5), 1, 2, 2),
    (2, 5, 4, 0, (9, 8), 1, 1, 2),
    (2, 3, 6, 2, (6, 7), 1, 2, 1),
    (3, 2, 3, 1, (3, 4, 5), 1, 2, 2),
    (3, 4, 3, 1, (3, 5, 4), 1, 2, 2),
    (4, 2, 3, 1, (2, 3, 2, 3), 1, 2, 2),
]


@pytest.mark.parametrize("N,S,G,pad,spatial,B,C,K", CASES)
def test_exact_nesting_equals_direct(N, S, G, pad, spatial, B, C, K):
    rng = random.Random(hash((N, S, G, pad)) & 0xffff)
    D = S + G - 1
    seq = ["0", "1", "-1", "2", "-2", "1/2", "-1/2", "3", "-3"]
    A_, B_, C_ = tc.synthesize(S, G, ",".join(seq[:D - 1] + ["inf"]))
    x = _rand_frac(rng, (B, C) + spatial)
    g = _rand_frac(rng, (K, C) + (G,) * N)
    y, st = wg.winograd_nd(x, g, (pad,) * N, A_, B_, C_, exact=True)
    ref = direct.direct_conv_py(x, g, pad)
    assert y.shape == ref.shape
    assert all(a == b for a, b in zip(y.reshape(-1), ref.reshape(-1)))


def test_tile_count_spec_example():
    out, tiles = wg.tile_geometry((7,), 3, 2, (0,))
    assert out == (5,) and tiles == (3,)


def test_paper_c3d_matrices_nest_exactly():
    # the paper's own F(4,3) C3D transforms in the 3-D nesting
    from tests.test_oracle_toomcook import _paper
    A_, B_, C_ = _paper("paper_c3d_f43.txt")
    rng = random.Random(5)
    x = _rand_frac(rng, (1, 2, 5, 4, 6))
    g = _rand_frac(rng, (2, 2, 3, 3, 3))
    y, _ = wg.winograd_nd(x, g, (1, 1, 1), A_, B_, C_, exact=True)
    ref = direct.direct_conv_py(x, g, 1)
    assert all(a == b for a, b in zip(y.reshape(-1), ref.reshape(-1)))


def test_2d_closed_form_matches_nmode():
    A_, B_, C_ = tc.synthesize(4, 3, "0,3/2,-3/2,2/3,-2/3,inf")
    rng = random.Random(9)
    d = _rand_frac(rng, (6, 6))
    gk = _rand_frac(rng, (3, 3))
    closed = wg.winograd_2d_closed_form(d, gk, A_, B_, C_, exact=True)
    nm = wg.multi_mode_product(
        wg.multi_mode_product(gk, wg.as_array(C_, True), [0, 1])
        * wg.multi_mode_product(d, wg.as_array(B_, True), [0, 1]),
        wg.as_array(A_, True), [0, 1])
    assert np.array_equal(closed, nm)
    # and it is the valid correlation of the 6x6 tile with the 3x3 kernel
    ref = direct.direct_conv_py(d[None, None], gk[None, None], 0)[0, 0]
    assert np.array_equal(closed, ref)


def test_nmode_unfolding_identity():
    # Y = X x_n U  <=>  Y_(n) = U X_(n)
    rng = np.random.default_rng(3)
    X = rng.standard_normal((3, 4, 5))
    U = rng.standard_normal((6, 4))
    Y = wg.nmode_product(X, U, 1)
    unfold = lambda T, n: np.moveaxis(T, n, 0).reshape(T.shape[n], -1)
    np.testing.assert_allclose(unfold(Y, 1), U @ unfold(X, 1), rtol=1e-13)


@pytest.mark.parametrize("N,S,pts,pad,spatial", [
    (2, 4, "0,3/2,-3/2,2/3,-2/3,inf", 1, (13, 11)),
    (2, 4, "0,1,-1,2,-2,inf", 1, (10, 9)),
    (3, 2, "0,1,-1,inf", 1, (5, 7, 6)),
    (3, 4, "0,3/2,-3/2,2/3,-2/3,inf", 1, (4, 9, 6)),
    (4, 2, "0,1,-1,inf", 1, (3, 4, 5, 4)),
])
def test_float64_winograd_vs_c_oracle(N, S, pts, pad, spatial):
    A_, B_, C_ = tc.synthesize(S, 3, pts)
    rng = np.random.default_rng(N + S)
    x = rng.standard_normal((2, 3) + spatial).astype(np.float32)
    g = rng.standard_normal((4, 3) + (3,) * N).astype(np.float32)
    y, _ = wg.winograd_nd(x, g, (pad,) * N, A_, B_, C_, exact=False)
    ref = direct.direct_conv_f64(x, g, pad)
    rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert rel < 1e-12


# per-axis transforms F(S_1 x .. x S_N, G_1 x .. x G_N) (Eq. (4) indexes B_n,
# C_n, A_n by axis): exact equality with the brute-force sum
PER_AXIS = [
    # N, S per axis, G per axis, pad, spatial, B, C, K
    (2, (2, 4), (3, 3), (1, 1), (5, 7), 1, 2, 2),       # F(2,3) x F(4,3)
    (2, (4, 2), (3, 3), (0, 1), (7, 4), 2, 1, 2),
    (2, (3, 2), (2, 3), (1, 0), (5, 6), 1, 2, 1),       # anisotropic kernel 2x3
    (2, (2, 3), (1, 3), (0, 1), (3, 5), 1, 2, 2),       # r = (1, 3): D_0 = 2, trivial kernel axis
    (3, (2, 4, 4), (3, 3, 3), (1, 1, 1), (3, 5, 4), 1, 2, 2),   # time F(2,3) x space F(4,3)
    (3, (1, 2, 3), (3, 2, 3), (1, 0, 1), (3, 3, 4), 1, 1, 2),
    (4, (2, 2, 3, 2), (3, 2, 2, 3), (1, 0, 0, 1), (2, 2, 3, 2), 1, 1, 1),
]


def _default_pts(S, G):
    seq = ["0", "1", "-1", "2", "-2", "1/2", "-1/2", "3", "-3"]
    D = S + G - 1
    return ",".join(seq[:D - 1] + ["inf"]) if D > 1 else "0"


@pytest.mark.parametrize("N,S,G,pad,spatial,B,C,K", PER_AXIS)
def test_per_axis_exact_equals_direct(N, S, G, pad, spatial, B, C, K):
    rng = random.Random(hash((N, S, G, pad)) & 0xffff)
    mats = [tc.synthesize(S[n], G[n], _default_pts(S[n], G[n])) for n in range(N)]
    A_, B_, C_ = ([m[i] for m in mats] for i in range(3))
    x = _rand_frac(rng, (B, C) + spatial)
    g = _rand_frac(rng, (K, C) + tuple(G))
    y, st = wg.winograd_nd(x, g, pad, A_, B_, C_, exact=True)
    ref = direct.direct_conv_py(x, g, pad)
    assert y.shape == ref.shape
    assert all(a == b for a, b in zip(y.ravel(), ref.ravel()))
    # P = prod D_n transform points, T = B prod ceil(out_n / S_n) tiles
    D = [S[n] + G[n] - 1 for n in range(N)]
    assert st["U"].shape == (int(np.prod(D)), C, K)
    assert st["V"].shape[1] == B * int(np.prod(st["tiles"]))


def test_per_axis_equal_axes_is_the_single_transform():
    rng = random.Random(7)
    A_, B_, C_ = tc.synthesize(2, 3, "0,1,-1,inf")
    x = _rand_frac(rng, (1, 2, 5, 4))
    g = _rand_frac(rng, (2, 2, 3, 3))
    y1, _ = wg.winograd_nd(x, g, (1, 1), A_, B_, C_, exact=True)
    y2, _ = wg.winograd_nd(x, g, (1, 1), [A_, A_], [B_, B_], [C_, C_], exact=True)
    assert all(a == b for a, b in zip(y1.ravel(), y2.ravel()))
