"""CPU-side checks of the C-ABI library (no GPU needed).

* libwino.so loads and exports every function include/wino.h declares.
* The product's host synthesis (C++, Vandermonde + Gauss-Jordan) agrees
  EXACTLY with the oracle's independent CRT construction (oracle/toomcook.py,
  Algorithm 1 of the paper) under the shared reading #6 normalisation, and
  passes the oracle's exact Eq. (1) identity check.
* Error codes of the argument validation.
"""
import re
from fractions import Fraction
from pathlib import Path

import pytest

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200 import wino
from oracle import toomcook as tc

ROOT = Path(__file__).resolve().parent.parent


def test_exports_match_header():
    header = (ROOT / "include" / "wino.h").read_text()
    declared = set(re.findall(r"\b(wino_[a-z_0-9]+)\s*\(", header))
    assert declared, "no declarations parsed"
    L = wino.lib()
    for name in declared:
        assert hasattr(L, name), "libwino.so does not export %s" % name
    assert declared == set(wino.EXPORTS)
    assert "sm_100a" in pkg.wino_version()


def _frac_matrix(rows):
    return [[Fraction(v) for v in row] for row in rows]


CASES = [(2, 3, None), (4, 3, None), (4, 3, "0,1,-1,2,-2,inf"), (2, 3, "0,1,-1,inf"),
         (3, 2, None), (3, 4, None), (5, 4, None), (4, 5, None), (3, 6, None), (2, 5, None),
         (6, 3, None), (1, 1, None), (1, 3, None), (2, 2, None),
         (4, 3, "0,1,-1,1/3,-1/3,inf"), (2, 3, "0,1/2,-3,inf"), (4, 3, "0,1,-1,2,-2,3")]


@pytest.mark.parametrize("m,r,points", CASES)
def test_host_synthesis_matches_oracle_exactly(m, r, points):
    d = pkg.wino_synthesize(m, r, points)
    AT, G, BT = _frac_matrix(d["AT"]), _frac_matrix(d["G"]), _frac_matrix(d["BT"])
    # exact Eq. (1) identity, checked by the oracle (paper orientation A, B, C)
    ok, why = tc.check_identity(AT, BT, G)
    assert ok, why
    # identical to the oracle's CRT construction for the same ordered points
    A_o, B_o, C_o = tc.synthesize(m, r, ",".join(d["points"]))
    assert AT == A_o and BT == B_o and G == C_o
    # doubles are the RNE images of the exact rationals
    for M, Mf in ((AT, d["AT_f64"]), (G, d["G_f64"]), (BT, d["BT_f64"])):
        for row, rowf in zip(M, Mf):
            assert [float(v) for v in row] == rowf


def test_default_points():
    assert pkg.wino_synthesize(2, 3)["points"] == ["0", "1", "-1", "inf"]
    assert pkg.wino_synthesize(4, 3)["points"] == ["0", "3/2", "-3/2", "2/3", "-2/3", "inf"]
    assert pkg.wino_synthesize(5, 4)["points"] == ["0", "1", "-1", "2", "-2", "1/2", "-1/2", "inf"]


@pytest.mark.parametrize("m,r,points,status", [
    (2, 3, "0,1,1,inf", wino.WINO_ERR_POINTS),
    (2, 3, "0,1,inf,inf", wino.WINO_ERR_POINTS),
    (2, 3, "0,1,-1", wino.WINO_ERR_POINTS),
    (2, 3, "0,1,x,inf", wino.WINO_ERR_POINTS),
    (0, 3, None, wino.WINO_ERR_ARG),
    (8, 8, None, wino.WINO_ERR_UNSUPPORTED),
])
def test_synthesis_errors(m, r, points, status):
    with pytest.raises(pkg.WinoError) as ei:
        pkg.wino_synthesize(m, r, points)
    assert ei.value.status == status
    assert pkg.wino_last_error()


def test_plan_argument_errors():
    cases = [
        (dict(N=5, dims=(4,) * 5), wino.WINO_ERR_ARG),
        (dict(N=2, dims=(2, 2), padding=(0, 0)), wino.WINO_ERR_SHAPE),
        (dict(N=2, dims=(8, 8), C=0), wino.WINO_ERR_ARG),
    ]
    for kw, status in cases:
        args = dict(N=2, dims=(8, 8), m=2, r=3, C=4, K=4, batch=1, padding=None)
        args.update(kw)
        with pytest.raises(pkg.WinoError) as ei:
            pkg.wino_plan_create_ex(args["N"], args["dims"], args["m"], args["r"], args["C"], args["K"],
                                    args["batch"], args["padding"])
        assert ei.value.status == status, pkg.wino_last_error()


def test_plan_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(pkg.WinoError) as ei:
        pkg.Plan(2, (8, 8), 2, 3, 4, 4, 1)
    assert ei.value.status in (wino.WINO_ERR_CUDA, wino.WINO_ERR_NOMEM)


def test_per_axis_plan_argument_errors():
    # wino_plan_create_nd validates before touching the device
    cases = [
        (dict(N=5, dims=(8,) * 5, m=(2,) * 5, r=(3,) * 5, padding=(1,) * 5), wino.WINO_ERR_ARG),
        (dict(m=(6, 2), r=(4, 3)), wino.WINO_ERR_UNSUPPORTED),     # alpha_0 = 9 > 8
        (dict(m=(2, 0), r=(3, 3)), wino.WINO_ERR_ARG),             # m_1 = 0
        (dict(dims=(2, 8), m=(2, 4), r=(3, 3), padding=(0, 1)), wino.WINO_ERR_SHAPE),   # kernel > input on axis 0
        (dict(C=0), wino.WINO_ERR_ARG),
    ]
    for kw, status in cases:
        args = dict(N=2, dims=(8, 8), m=(2, 4), r=(3, 3), C=4, K=4, batch=1, padding=(1, 1))
        args.update(kw)
        with pytest.raises(pkg.WinoError) as ei:
            pkg.wino_plan_create_nd(args["N"], args["dims"], args["m"], args["r"], args["C"], args["K"],
                                    args["batch"], args["padding"])
        assert ei.value.status == status, pkg.wino_last_error()
