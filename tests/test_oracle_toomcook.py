"""Pins for oracle.toomcook (exact synthesis of A, B, C).

Pinned against the paper's printed matrices, its
worked F(2,3) example and minimal algorithm, Table 1
(PAPER.md:276-289), the SPEC polynomial examples, and a perturbation test.
"""
import random
from fractions import Fraction as F

import pytest

from oracle import toomcook as tc
from tests.conftest import read_golden


def _paper(name):
    d = read_golden(name)
    A, B = d["A"], d["B"]
    C = d["C"] if "C" in d else [list(col) for col in zip(*d["CT"])]
    return A, B, C


# ---------------------------------------------------------------- polynomials
def test_poly_examples():
    assert tc.poly_mul([1, 1], [1, -1]) == [1, 0, -1]
    assert tc.poly_mul([1, 2], []) == []
    assert tc.poly_mul([1, 1, 1], [1, 2, 3, 4])[2] == 6
    assert tc.poly_divmod([-1, 0, 1], [-1, 1]) == ([1, 1], [])
    assert tc.poly_divmod([0, 0, 0, 1], [0, 1]) == ([0, 0, 1], [])
    assert tc.poly_divmod([1, 0, 1], [-2, 1]) == ([2, 1], [5])
    with pytest.raises(ZeroDivisionError):
        tc.poly_divmod([1], [])


def test_crt_basis_examples():
    a = tc.crt_basis([[0, 1], [-1, 1]])                                 # {x, x-1} S:80
    assert a == [[1, -1], [0, 1]]
    assert tc.crt_basis([[0, 1]]) == [[1]]
    with pytest.raises(ValueError):
        tc.crt_basis([[0, 1], [0, 1]])


def test_algorithm1_equals_product():
    rng = random.Random(0)
    pts = [0, 1, -1, 2, -2, 3, F(1, 2)]
    for _ in range(20):
        g = [F(rng.randint(-9, 9), rng.randint(1, 5)) for _ in range(rng.randint(1, 4))]
        d = [F(rng.randint(-9, 9), rng.randint(1, 5)) for _ in range(rng.randint(1, 4))]
        moduli = [[-F(p), 1] for p in pts]
        assert tc.fast_vector_convolve_crt(g, d, moduli) == tc.poly_mul(g, d)
    # g=(1,1,1), d=(1,2,3,4), points {0,1,-1,2,-2,3}
    mod = [[-F(p), 1] for p in (0, 1, -1, 2, -2, 3)]
    assert tc.fast_vector_convolve_crt([1, 1, 1], [1, 2, 3, 4], mod) == tc.poly_mul([1, 1, 1], [1, 2, 3, 4])
    with pytest.raises(ValueError):
        tc.fast_vector_convolve_crt([1, 1, 1], [1, 2, 3, 4], mod[:3])


# ------------------------------------------------------------ paper matrices
def test_paper_f23_passes_identity():
    ok, why = tc.check_identity(*_paper("paper_f23.txt"))
    assert ok, why


def test_paper_c3d_f43_passes_identity():
    ok, why = tc.check_identity(*_paper("paper_c3d_f43.txt"))
    assert ok, why


@pytest.mark.parametrize("which,i,j", [("A", 1, 2), ("B", 3, 3), ("C", 1, 0), ("A", 0, 0)])
def test_perturbation_detected(which, i, j):
    A, B, C = _paper("paper_f23.txt")
    M = {"A": A, "B": B, "C": C}[which]
    M[i][j] += F(1, 7)
    ok, why = tc.check_identity(A, B, C)
    assert not ok and why is not None and why[3] != why[4]


def test_worked_example_values():
    w = read_golden("worked_f23.txt")
    A, B, C = _paper("paper_f23.txt")
    g, d = w["g"][0], w["d"][0]
    Cg = [sum(r[j] * g[j] for j in range(3)) for r in C]
    Bd = [sum(r[j] * d[j] for j in range(4)) for r in B]
    assert Cg == w["Cg"][0] and Bd == w["Bd"][0]
    assert [a * b for a, b in zip(Cg, Bd)] == w["prod"][0]
    assert tc.apply_eq1(A, B, C, g, d) == w["s"][0]
    assert tc.correlate_valid(d, g) == w["s"][0]
    # minimal algorithm of
    d0, d1, d2, d3 = d
    g0, g1, g2 = g
    m = [(d0 - d2) * g0, (d1 + d2) * (g0 + g1 + g2) / 2, (d2 - d1) * (g0 - g1 + g2) / 2, (d1 - d3) * g2]
    assert m == w["m"][0]
    assert [m[0] + m[1] + m[2], m[1] - m[2] - m[3]] == w["s"][0]


def _diag_equivalent(P, Q):
    """(A,B,C) triples equal up to per-point scaling a_k b_k c_k = 1
    (A unique only up to diagonal rescaling)."""
    (Ap, Bp, Cp), (Aq, Bq, Cq) = P, Q
    D = len(Bp)
    for k in range(D):
        def ratio(u, v):
            r = None
            for a, b in zip(u, v):
                if (a == 0) != (b == 0):
                    return None
                if a != 0:
                    if r is None:
                        r = a / b
                    elif a / b != r:
                        return None
            return r
        ra = ratio([row[k] for row in Ap], [row[k] for row in Aq])
        rb = ratio(Bp[k], Bq[k])
        rc = ratio(Cp[k], Cq[k])
        if None in (ra, rb, rc) or ra * rb * rc != 1:
            return False
    return True


def test_synthesis_reproduces_paper_f23():
    ours = tc.synthesize(2, 3, "0,1,-1,inf")
    assert _diag_equivalent(_paper("paper_f23.txt"), ours)


def test_synthesis_reproduces_paper_c3d():
    # points read off A's columns: 0, 1, -1, 1/3, -1/3, inf
    ours = tc.synthesize(4, 3, "0,1,-1,1/3,-1/3,inf")
    assert _diag_equivalent(_paper("paper_c3d_f43.txt"), ours)


def test_normalization_puts_denominators_in_C():
    A, B, C = tc.synthesize(2, 3, "0,1,-1,inf")
    ref_A, ref_B, ref_C = _paper("paper_f23.txt")
    assert C[1] == ref_C[1] and C[2] == ref_C[2]           # (1/2,1/2,1/2), (1/2,-1/2,1/2)
    assert all(v.denominator == 1 for row in B for v in row)


@pytest.mark.parametrize("S,G", [(2, 3), (3, 2), (4, 3), (3, 4), (5, 4), (4, 5), (3, 6), (2, 5),
                                 (6, 3), (1, 1), (1, 3), (2, 2)])
def test_synthesis_identity_exact(S, G):
    D = S + G - 1
    seq = ["0", "1", "-1", "2", "-2", "1/2", "-1/2", "3", "-3"]
    pts = ["0"] if D == 1 else seq[:D - 1] + ["inf"]
    ok, why = tc.check_identity(*tc.synthesize(S, G, ",".join(pts)))
    assert ok, why
    # without a point at infinity too (all finite)
    ok, why = tc.check_identity(*tc.synthesize(S, G, ",".join(seq[:D])))
    assert ok, why


def test_alt_points_identity():
    ok, why = tc.check_identity(*tc.synthesize(4, 3, "0,3/2,-3/2,2/3,-2/3,inf"))
    assert ok, why


def test_bad_points_rejected():
    with pytest.raises(ValueError):
        tc.synthesize(2, 3, "0,1,1,inf")
    with pytest.raises(ValueError):
        tc.synthesize(2, 3, "0,1,inf,inf")
    with pytest.raises(ValueError):
        tc.synthesize(2, 3, "0,1,-1")


def test_table1():
    for row in read_golden("table1.txt")["row"]:
        _, D, G, S, sa, sb, sc, s2, s3, pts = row
        pts = pts.split("=", 1)[1]
        A, B, C = tc.synthesize(int(S), int(G), pts)
        assert len(B) == D
        assert round(tc.sparsity(A), 2) == float(sa)
        assert round(tc.sparsity(B), 2) == float(sb)
        assert round(tc.sparsity(C), 2) == float(sc)
        # (SG/D)^N rounded half up to 2 decimals (15.625 -> 15.63)
        half_up = lambda v: float(F(round(F(v) * 1000)) // 10 + (1 if round(F(v) * 1000) % 10 >= 5 else 0)) / 100
        assert half_up((F(S) * G / D) ** 2) == float(s2)
        assert half_up((F(S) * G / D) ** 3) == float(s3)
