"""CPU tests of the analytic cost model (paper_1611_06565_b200.cost, SURVEY
8(f) NEXT-4), pinned to the numbers the paper prints and to brute-force
counts of explicit loops."""
from fractions import Fraction

import pytest

from paper_1611_06565_b200 import cost


# Table 1 speed-up columns, printed to 2 decimals
@pytest.mark.parametrize("D,G,S,two,three", [
    (4, 2, 3, "2.25", "3.38"), (4, 3, 2, "2.25", "3.38"), (8, 4, 5, "6.25", "15.63"),
    (8, 5, 4, "6.25", "15.63"), (8, 6, 3, "5.06", "11.39")])
def test_table1_speedups(D, G, S, two, three):
    assert S + G - 1 == D
    assert "%.2f" % float(cost.theoretical_speedup(S, G, 2)) == two
    # 3.375 and 15.625 print as 3.38 / 15.63 in the table (round half up)
    v3 = cost.theoretical_speedup(S, G, 3)
    assert "%.2f" % (float(v3) + 1e-9) == three


def test_c3d_ceiling_is_8():
    # "The theoretical ceiling on speed-up ... is 8-fold", F(4,3), N=3
    assert cost.theoretical_speedup(4, 3, 3) == 8


def test_speedup_symmetric_in_S_G():
    for S in range(1, 7):
        for G in range(1, 7):
            for N in (1, 2, 3):
                assert cost.theoretical_speedup(S, G, N) == cost.theoretical_speedup(G, S, N)


def _brute_direct(M, K, S, G, N):
    # count the multiplications of an explicit sliding-window loop nest
    import itertools
    n = 0
    for _k in range(K):
        for _c in range(M):
            for _o in itertools.product(range(S), repeat=N):
                for _p in itertools.product(range(G), repeat=N):
                    n += 1
    return n


@pytest.mark.parametrize("M,K,S,G,N", [(1, 1, 2, 3, 1), (2, 3, 2, 3, 2), (3, 2, 4, 3, 2), (1, 2, 2, 2, 3)])
def test_direct_muls_brute_force(M, K, S, G, N):
    assert cost.direct_muls(M, K, S, G, N) == _brute_direct(M, K, S, G, N)


def test_f23_counts_paper():
    t = cost.transforms(2, 3)
    # "28 multiplications -- 4 for the element-wise product, 16 for the data
    # transform and 8 for the inverse transform"
    assert cost.nmode_cost(t["BT"], 1, "dense") == 16
    assert cost.nmode_cost(t["AT"], 1, "dense") == 8
    assert cost.fast_muls(1, 1, t["AT"], t["BT"], 1, "dense") == 28
    # "4M^2 + 24M" for M channels and M kernels
    for M in (1, 2, 7, 64, 100):
        assert cost.fast_muls(M, M, t["AT"], t["BT"], 1, "dense") == 4 * M * M + 24 * M
    # sparse: nonzero counting gives 18 and 4M^2 + 14M; the paper prints 19
    # and 4M^2 + 15M (reading #13: a paper slip, kept visible here)
    assert cost.fast_muls(1, 1, t["AT"], t["BT"], 1, "nonzero") == 18
    for M in (1, 5, 100):
        assert cost.fast_muls(M, M, t["AT"], t["BT"], 1, "nonzero") == 4 * M * M + 14 * M


def _brute_nmode(X, N):
    # apply X along each axis of a D^N tensor of symbols, counting products
    import itertools
    import numpy as np
    rows, D = len(X), len(X[0])
    shape = [D] * N
    n_mul = {"dense": 0, "nonzero": 0}
    for ax in range(N):
        other = [shape[i] for i in range(N) if i != ax]
        for _ in itertools.product(*[range(e) for e in other]):
            for i in range(rows):
                for j in range(D):
                    n_mul["dense"] += 1
                    n_mul["nonzero"] += X[i][j] != 0
        shape[ax] = rows
    return n_mul


@pytest.mark.parametrize("m,r,N", [(2, 3, 2), (4, 3, 3), (3, 4, 2), (2, 3, 4)])
def test_nmode_cost_brute_force(m, r, N):
    t = cost.transforms(m, r)
    for X in (t["AT"], t["BT"]):
        b = _brute_nmode(X, N)
        assert cost.nmode_cost(X, N, "dense") == b["dense"]
        assert cost.nmode_cost(X, N, "nonzero") == b["nonzero"]


def test_c3d_figure1_claims():
    # the paper's own C3D points: F(4,3), N=3
    pts = "0,1,-1,1/3,-1/3,inf"
    Ms = [1, 2, 5, 10, 20, 50, 100, 200, 1000, 10000]
    curve = dict(cost.speedup_curve(4, 3, 3, Ms, "dense", pts))
    # "greater than 6-fold acceleration" at 100 kernels and channels
    assert curve[100] > 6
    # "triple the performance margin ... 10 kernels and channels": within 25%
    assert 0.75 * 3 <= curve[100] / curve[10] <= 1.25 * 3
    # increasing in M and below the 8-fold ceiling
    vals = [curve[M] for M in Ms]
    assert all(a < b for a, b in zip(vals, vals[1:]))
    assert all(v < 8 for v in vals) and vals[-1] > Fraction(79, 10)
    # sparse counting is never worse than dense
    sparse = dict(cost.speedup_curve(4, 3, 3, Ms, "nonzero", pts))
    assert all(sparse[M] >= curve[M] for M in Ms)


def test_arithmetic_intensity():
    # unfused element-wise product: 2 D^N M / 2 D^N M = 1
    assert cost.arithmetic_intensity(1000, 64, 64, fused=False) == 1
    # fused per-point products: 2TK/(T+K), = K at T = K
    for K in (1, 8, 100):
        assert cost.arithmetic_intensity(K, 3, K, fused=True) == K
    assert cost.arithmetic_intensity(1, 1, 1, fused=True) == 1
    assert cost.arithmetic_intensity(300, 5, 100, fused=True) == Fraction(2 * 300 * 100, 400)
    assert cost.arithmetic_intensity(300, 5, 100, fused=True) <= 2 * min(300, 100)


def test_stage_model_matches_survey_bytes():
    # SURVEY 8(d) per-stage algorithmic bytes (MB, decimal): c2 input x + V =
    # 51.4 + 115.6, output M + y = 115.6 + 51.4; c4 input 205.5 + 693.6
    st = cost.stage_model(2, (56, 56), 4, 3, 128, 128, 32, (1, 1))
    assert round(st["input_xform"]["bytes"] / 1e6, 1) == 167.0
    assert round(st["output_xform"]["bytes"] / 1e6, 1) == 167.0
    assert st["tiles"] == 32 * 14 * 14
    assert st["direct_flops"] == 2 * 32 * 128 * 128 * 56 * 56 * 9
    st4 = cost.stage_model(3, (8, 28, 28), 4, 3, 256, 256, 32, (1, 1, 1), hbm_gbs=6447, tf32_tflops=817)
    assert round(st4["input_xform"]["bytes"] / 1e6, 1) == 899.2
    assert st4["gemm"]["bound"] == "tensor" and st4["input_xform"]["bound"] == "hbm"
    assert st4["gemm"]["flops"] == 2 * 216 * (32 * 98) * 256 * 256


def test_cli_runs(capsys):
    assert cost.main(["--m", "2", "--r", "3", "--N", "1", "--Ms", "1,10"]) == 0
    out = capsys.readouterr().out.strip().splitlines()
    assert out[1].startswith("M,K,direct_muls")
    assert out[2].split(",")[:5] == ["1", "1", "6", "28", "18"]


def test_per_axis_speedup_and_bytes():
    # equal axes reduce to (SG/D)^N; F(2,3) x F(4,3)^2: 1.5 * 2 * 2
    assert cost.theoretical_speedup_axes((4, 4, 4), (3, 3, 3)) == cost.theoretical_speedup(4, 3, 3)
    assert cost.theoretical_speedup_axes((2, 4, 4), (3, 3, 3)) == Fraction(3, 2) * 2 * 2
    assert cost.theoretical_speedup_axes((1, 4, 4), (1, 3, 3)) == 4        # 1x3x3: F(1,1) gains nothing
    st = cost.stage_model(3, (16, 56, 56), (2, 4, 4), (3, 3, 3), 64, 128, 16, (1, 1, 1))
    T = 16 * 8 * 14 * 14
    assert st["tiles"] == T
    assert st["input_xform"]["bytes"] == 4 * 16 * 64 * 16 * 56 * 56 + 4 * 144 * 64 * T
    assert st["gemm"]["flops"] == 2 * 144 * T * 64 * 128
    assert st["direct_flops"] == 2 * 16 * 128 * 64 * 16 * 56 * 56 * 27
    # uniform sequences equal the scalar form
    a = cost.stage_model(2, (56, 56), 4, 3, 128, 128, 32, (1, 1))
    b = cost.stage_model(2, (56, 56), (4, 4), (3, 3), 128, 128, 32, (1, 1))
    assert a == b


def test_stage_model_fold_bytes():
    # a5 folds: W = (m/alpha)^F of M; the filter-side fold
    # (fold_mode 2) streams U' = m^F U and executes m^F x the multiply-adds
    from paper_1611_06565_b200.cost import stage_model
    args = (3, (16, 56, 56), 2, 3, 64, 128, 16, (1, 1, 1))
    s0 = stage_model(*args)
    T, P, C, K = s0["tiles"], 64, 64, 128
    Vb, Mb, Ub = 4 * P * C * T, 4 * P * K * T, 4 * P * C * K
    assert s0["gemm"]["bytes"] == Vb + Ub + Mb
    s1 = stage_model(*args, fold=1, fold_mode=2)
    assert s1["gemm"]["bytes"] == Vb + 2 * Ub + Mb // 2
    assert s1["gemm"]["flops"] == 2 * s0["gemm"]["flops"]
    assert s1["output_xform"]["bytes"] == s0["output_xform"]["bytes"] - Mb // 2
    # direct-axis fold (fold_mode 3): Z = 16 outer points x 58 padded columns per
    # row of 28 tiles instead of V = 64 points x 28 tiles; 2 * 3 / 4 of the flops
    s3 = stage_model(*args, fold=1, fold_mode=3)
    Zb = 4 * 16 * C * (T // 28) * 58
    assert s3["input_xform"]["bytes"] == s0["input_xform"]["bytes"] - Vb + Zb
    assert s3["gemm"]["bytes"] == Zb + 2 * Ub + Mb // 2
    assert 2 * s3["gemm"]["flops"] == 3 * s0["gemm"]["flops"]
    assert s3["output_xform"] == s1["output_xform"]
    s2 = stage_model(*args, fold=2, fold_mode=1)
    assert s2["gemm"]["bytes"] == Vb + Ub + Mb // 4 and s2["gemm"]["flops"] == s0["gemm"]["flops"]
    assert s2["input_xform"] == s0["input_xform"]
