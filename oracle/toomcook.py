"""oracle.toomcook -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Exact-rational synthesis of the 1-D fast-convolution transforms of Eq. (1)
(PAPER.md:52-56), s = A [(C g) (.) (B d)], following the paper's
construction step by step:

* Theorem 1 / Algorithm 1: residues of g(x), d(x) modulo
  pairwise-coprime moduli m^(k)(x), residue products, CRT recombination
  s(x) = sum_k s^(k)(x) a^(k)(x).  With linear moduli m^(k) = x - p_k the
  residue of a polynomial is its value at p_k ("C and B are the
  remainders of the polynomial divisions g(x) and d(x) by m^(k)(x)"); the
  "point at infinity" supplies the product of leading coefficients (reading
  #5 of DESIGN.md; SPEC.md:138 homogeneous treatment).
* This gives the linear convolution of a length-G kernel with a length-S data
  vector, length D = S + G - 1.  The F(S,G) algorithm of
  Eq. (1), whose matrices the paper prints and which
  computes a *correlation* over a length-D tile (reading #1), is its
  transpose: A = E_S^T, C = E_G, B = Lambda^T, where E_n are the residue
  (evaluation) matrices and Lambda the CRT recombination matrix.
* Reading #6 (diagonal scaling): each row of B is scaled to a primitive
  integer vector with a positive factor, the inverse factor multiplied into
  the matching row of C ("denominators in C/G").

All arithmetic is ``fractions.Fraction``.  Notation follows the paper:
A is S x D, B is D x D, C is D x G.  (The product code calls these
A^T (m x alpha), B^T, G; same matrices.)
"""
from __future__ import annotations

from fractions import Fraction
from functools import reduce
from math import gcd
from typing import List, Sequence, Tuple, Union

INF = "inf"
Point = Union[Fraction, str]
Poly = List[Fraction]          # coefficients, lowest degree first; [] is zero


# ----------------------------------------------------------------- polynomials
def _trim(p: Sequence[Fraction]) -> Poly:
    p = [Fraction(c) for c in p]
    while p and p[-1] == 0:
        p.pop()
    return p


def poly_mul(p: Sequence, q: Sequence) -> Poly:
    """Coefficient i of p*q is sum_k p_k q_{i-k}."""
    p, q = _trim(p), _trim(q)
    if not p or not q:
        return []
    out = [Fraction(0)] * (len(p) + len(q) - 1)
    for i, a in enumerate(p):
        for j, b in enumerate(q):
            out[i + j] += a * b
    return _trim(out)


def poly_add(p: Sequence, q: Sequence) -> Poly:
    n = max(len(p), len(q))
    return _trim([(Fraction(p[i]) if i < len(p) else 0) + (Fraction(q[i]) if i < len(q) else 0)
                  for i in range(n)])


def poly_divmod(p: Sequence, m: Sequence) -> Tuple[Poly, Poly]:
    """p = q m + r with deg r < deg m (Algorithm 1 step (1))."""
    p, m = _trim(p), _trim(m)
    if not m:
        raise ZeroDivisionError("division by zero polynomial")
    r = list(p)
    q = [Fraction(0)] * max(len(p) - len(m) + 1, 0)
    while len(r) >= len(m) and r:
        shift = len(r) - len(m)
        coef = r[-1] / m[-1]
        q[shift] = coef
        for i, mc in enumerate(m):
            r[shift + i] -= coef * mc
        r = _trim(r)
    return _trim(q), r


def poly_egcd(a: Sequence, b: Sequence) -> Tuple[Poly, Poly, Poly]:
    """Extended Euclid over Q[x]: returns (g, s, t) with s a + t b = g."""
    r0, r1 = _trim(a), _trim(b)
    s0, s1 = [Fraction(1)], []
    t0, t1 = [], [Fraction(1)]
    while r1:
        q, r = poly_divmod(r0, r1)
        r0, r1 = r1, r
        s0, s1 = s1, poly_add(s0, [-c for c in poly_mul(q, s1)])
        t0, t1 = t1, poly_add(t0, [-c for c in poly_mul(q, t1)])
    return r0, s0, t0


def crt_basis(moduli: Sequence[Sequence]) -> List[Poly]:
    """Recombinators a^(k) with a^(k) = 1 mod m^(k), 0 mod m^(j), j != k
    (Theorem 1; Algorithm 1 step (3))."""
    moduli = [_trim(m) for m in moduli]
    M = reduce(poly_mul, moduli, [Fraction(1)])
    out = []
    for k, mk in enumerate(moduli):
        Mk, rem = poly_divmod(M, mk)
        assert not rem
        g, s, _ = poly_egcd(Mk, mk)
        if len(g) != 1:
            raise ValueError("moduli %d and another are not coprime" % k)
        # s*Mk = g (mod mk) with g a nonzero constant
        a = poly_mul([c / g[0] for c in s], Mk)
        out.append(poly_divmod(a, M)[1])
    return out


def fast_vector_convolve_crt(g: Sequence, d: Sequence, moduli: Sequence[Sequence]) -> Poly:
    """Algorithm 1 verbatim: residues, residue products,
    recombination; requires deg m(x) > deg(g d) (Theorem 1 proviso)."""
    M = reduce(poly_mul, [_trim(m) for m in moduli], [Fraction(1)])
    g, d = _trim(g), _trim(d)
    if g and d and len(M) - 1 <= (len(g) - 1) + (len(d) - 1):
        raise ValueError("modulus degree too small")
    a = crt_basis(moduli)
    s = []
    for mk, ak in zip(moduli, a):
        gk = poly_divmod(g, mk)[1]                  # (1) residues
        dk = poly_divmod(d, mk)[1]
        sk = poly_divmod(poly_mul(gk, dk), mk)[1]   # (2) residue product
        s = poly_add(s, poly_mul(sk, ak))           # (3) recombination
    return poly_divmod(s, M)[1]


# ------------------------------------------------------------------ points
def parse_points(spec: Union[str, Sequence]) -> List[Point]:
    """'0,1,-1,inf' / '3/2' / sequence -> list of Fraction or INF."""
    items = spec.split(",") if isinstance(spec, str) else list(spec)
    out: List[Point] = []
    for it in items:
        s = str(it).strip().lower()
        out.append(INF if s in ("inf", "infinity", "oo") else Fraction(s))
    return out


def _check_points(points: Sequence[Point], D: int) -> None:
    if len(points) != D:
        raise ValueError("need exactly D = S + G - 1 = %d points, got %d" % (D, len(points)))
    if sum(1 for p in points if p == INF) > 1:
        raise ValueError("more than one point at infinity")
    fin = [p for p in points if p != INF]
    if len(set(fin)) != len(fin):
        raise ValueError("duplicate points")


# -------------------------------------------------------------- synthesis
def residue_matrix(points: Sequence[Point], n: int) -> List[List[Fraction]]:
    """E_n (D x n): row k holds the residues of the monomials x^0..x^{n-1}
    modulo m^(k)(x) = x - p_k, i.e. Algorithm 1 step (1) applied to a basis
    (computed by actual polynomial division); the infinity row selects the
    leading (x^{n-1}) coefficient."""
    rows = []
    for p in points:
        if p == INF:
            rows.append([Fraction(int(j == n - 1)) for j in range(n)])
        else:
            row = []
            for j in range(n):
                mono = [Fraction(0)] * j + [Fraction(1)]
                r = poly_divmod(mono, [-p, Fraction(1)])[1]
                row.append(r[0] if r else Fraction(0))
            rows.append(row)
    return rows


def recombination_matrix(points: Sequence[Point]) -> List[List[Fraction]]:
    """Lambda (D x D): column k = coefficients of the CRT recombinator a^(k)
    (Algorithm 1 step (3)).  With a point at infinity the finite moduli have
    product M(x) of degree D-1 and s(x) = [sum_k s^(k) a^(k)] mod M + s_inf M(x),
    so the infinity column is M(x)'s coefficient vector."""
    D = len(points)
    fin = [p for p in points if p != INF]
    moduli = [[-p, Fraction(1)] for p in fin]
    a = crt_basis(moduli) if moduli else []
    M = reduce(poly_mul, moduli, [Fraction(1)])
    cols, fi = [], 0
    for p in points:
        if p == INF:
            col = M
        else:
            col = a[fi]
            fi += 1
        cols.append(list(col) + [Fraction(0)] * (D - len(col)))
    return [[cols[k][i] for k in range(D)] for i in range(D)]


def synthesize(S: int, Gk: int, points: Sequence[Point], normalize: bool = True):
    """(A, B, C) of Eq. (1) for F(S, G) from D = S+G-1 points.

    Linear convolution (kernel length G, data length S) by Algorithm 1 is
    s = Lambda [(E_G g) (.) (E_S d)]; its transpose is the correlation
    F(S,G): A = E_S^T (S x D), C = E_G (D x G), B = Lambda^T (D x D).
    """
    D = S + Gk - 1
    points = parse_points(points) if isinstance(points, str) else list(points)
    _check_points(points, D)
    ES = residue_matrix(points, S)
    EG = residue_matrix(points, Gk)
    Lam = recombination_matrix(points)
    A = [[ES[k][i] for k in range(D)] for i in range(S)]
    C = [list(row) for row in EG]
    B = [[Lam[j][i] for j in range(D)] for i in range(D)]
    if normalize:
        B, C = normalize_denominators(B, C)
    return A, B, C


def normalize_denominators(B, C):
    """Reading #6: row k of B -> primitive integer vector (positive factor
    lambda_k), row k of C multiplied by lambda_k; (C g)(.)(B d) unchanged."""
    B2, C2 = [], []
    for brow, crow in zip(B, C):
        L = reduce(lambda a, b: a * b // gcd(a, b), [f.denominator for f in brow], 1)
        ints = [int(f * L) for f in brow]
        h = reduce(gcd, [abs(v) for v in ints], 0) or 1
        lam = Fraction(h, L)
        B2.append([f / lam for f in brow])
        C2.append([f * lam for f in crow])
    return B2, C2


# ------------------------------------------------------------ validation
def correlate_valid(d: Sequence, g: Sequence) -> list:
    """Valid cross-correlation s_o = sum_k g_k d_{o+k} (PAPER.md:139, 1-D)."""
    n = len(d) - len(g) + 1
    return [sum((g[k] * d[o + k] for k in range(len(g))), Fraction(0)) for o in range(n)]


def apply_eq1(A, B, C, g, d) -> list:
    """s = A [(C g) (.) (B d)] (Eq. (1)) in exact arithmetic."""
    Cg = [sum((row[j] * g[j] for j in range(len(g))), Fraction(0)) for row in C]
    Bd = [sum((row[j] * d[j] for j in range(len(d))), Fraction(0)) for row in B]
    prod = [a * b for a, b in zip(Cg, Bd)]
    return [sum((row[j] * prod[j] for j in range(len(prod))), Fraction(0)) for row in A]


def check_identity(A, B, C):
    """Exact check of the Eq. (1) identity on every basis pair (g=e_i, d=e_j):
    the bilinear map A[(Cg)(.)(Bd)] equals valid correlation iff it does on a
    basis.  Returns (ok, first_violation or None) with violation =
    (i, j, output o, got, expected)."""
    S, D, Gk = len(A), len(B), len(C[0])
    if any(len(r) != D for r in A) or any(len(r) != D for r in B) or len(C) != D:
        raise ValueError("dimension mismatch among A, B, C")
    if S + Gk - 1 != D:
        raise ValueError("D != S + G - 1")
    for i in range(Gk):
        g = [Fraction(int(t == i)) for t in range(Gk)]
        for j in range(D):
            d = [Fraction(int(t == j)) for t in range(D)]
            got = apply_eq1(A, B, C, g, d)
            exp = correlate_valid(d, g)
            for o in range(S):
                if got[o] != exp[o]:
                    return False, (i, j, o, got[o], exp[o])
    return True, None


def sparsity(Mx) -> float:
    """Fraction of exactly-zero entries (Table 1)."""
    flat = [v for row in Mx for v in row]
    return sum(1 for v in flat if v == 0) / len(flat)
