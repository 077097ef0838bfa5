"""GPU parity of the a5 filter-side fold (fold_mode 2, kernels.h UFoldTab):
A^T of the F innermost axes multiplied into the cached transformed filter
U'[xo][(q,c)][(o,k)] = A^T_F[o][q] U_{xo*Q+q}[c][k], the GEMM run as one
plain GEMM per outer point over V viewed as [P/Q][Q*C][T], a4 on the outer
axes ("the inverse transform can be applied once over the
reduced output"; Eq. (4)-(5)).  Every output of ragged
shrunken configs against the float64 direct oracle at BASELINE.json's
tolerances, in both GEMM schemes; W against the oracle's S_hat contracted
with A^T; full-size configs sampled."""
import numpy as np
import pytest
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, LayerConfig, make_inputs, tolerance
from oracle import direct, fp32model as fm, toomcook as tc, winograd as wg

pytestmark = pytest.mark.gpu

# ragged: partial channel chunks (C not a multiple of 32), K not a multiple
# of the N tile, partial edge tiles, T not a multiple of 128
UF_SMALL = {
    "c3": LayerConfig("u3s", 3, 2, 40, 48, (5, 13, 11), 3, 1, 2, "normal", "he"),
    "c5": LayerConfig("u5s", 4, 2, 36, 20, (3, 4, 5, 6), 3, 1, 2, "normal", "he"),
    "c2": LayerConfig("u2s", 2, 2, 32, 40, (29, 23), 3, 1, 4, "normal", "he"),
}
CASES = [("c3", 1), ("c2", 1)]
SCHEMES = {"3xf16": "4", "3xtf32": "3"}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _plan(cfg, F, scheme, monkeypatch, batch):
    monkeypatch.setenv("WINO_UFOLD", str(F))
    monkeypatch.setenv("WINO_DFOLD", "0")   # the plain filter-side fold (the direct-axis fold: test_gpu_dfold.py)
    monkeypatch.setenv("WINO_FOLD", "0")
    monkeypatch.setenv("WINO_GEMM_AUTO_MODE", SCHEMES[scheme])
    return pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, batch, cfg.padding)


def _run(cfg, F, scheme, monkeypatch, x, g, bias=None, relu=False):
    plan = _plan(cfg, F, scheme, monkeypatch, x.shape[0])
    info = plan.info
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda(), bias=bias, relu=relu).cpu()
    plan.close()
    return y, info


@pytest.mark.parametrize("scheme", list(SCHEMES))
@pytest.mark.parametrize("name,F", CASES)
def test_ufold_small_every_output(name, F, scheme, monkeypatch):
    cfg = UF_SMALL[name]
    x, g = make_inputs(cfg)
    y, info = _run(cfg, F, scheme, monkeypatch, x, g)
    assert info["fold"] == F and info["fold_mode"] == 2, info
    assert info["gemm_mode"] == int(SCHEMES[scheme]), info
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
    rel, mx = fm.errors(y.double().numpy(), ref)
    tl, tm = tolerance(cfg)
    print("%s ufold F=%d %s relL2=%.3e max=%.3e" % (cfg.name, F, scheme, rel, mx))
    assert rel <= tl and mx <= tm


@pytest.mark.parametrize("name,F", [("c3", 1), ("c2", 1)])
def test_ufold_bias_relu(name, F, monkeypatch):
    cfg = UF_SMALL[name]
    x, g = make_inputs(cfg)
    b = torch.randn(cfg.K, generator=torch.Generator().manual_seed(5))
    y, _ = _run(cfg, F, "3xf16", monkeypatch, x, g)
    yb, _ = _run(cfg, F, "3xf16", monkeypatch, x, g, bias=b.cuda(), relu=True)
    shape = (1, cfg.K) + (1,) * cfg.N
    assert torch.equal(yb, torch.clamp_min(y + b.view(shape), 0.0))


@pytest.mark.parametrize("name,F", [("c3", 1)])
def test_ufold_full_size_sampled(name, F, monkeypatch):
    cfg = CONFIGS[name]
    x, g = make_inputs(cfg)
    y, info = _run(cfg, F, "3xf16", monkeypatch, x, g)
    assert info["fold"] == F and info["fold_mode"] == 2
    rng = np.random.default_rng(7)
    n = y.numel()
    idx = np.concatenate([np.arange(64), np.arange(n - 64, n), rng.integers(0, n, 4096)])
    ref = direct.direct_conv_at(x.numpy(), g.numpy(), cfg.pad, idx)
    rel, mx = fm.errors(y.reshape(-1)[torch.from_numpy(idx)].double().numpy(), ref)
    tl, tm = tolerance(cfg)
    print("%s full ufold F=%d relL2=%.3e max=%.3e" % (name, F, rel, mx))
    assert rel <= tl and mx <= tm


@pytest.mark.parametrize("scheme", list(SCHEMES))
@pytest.mark.parametrize("name,F", [("c3", 1)])
def test_ufold_stage_w(name, F, scheme, monkeypatch):
    """W (the GEMM's output, in the M workspace) against the oracle: S_hat of
    Eq. (5) with A^T applied along the last F axes (Eq. (4)); the same array
    the epilogue fold writes (tests/test_gpu_fold.py)."""
    cfg = UF_SMALL[name]
    x, g = make_inputs(cfg)
    plan = _plan(cfg, F, scheme, monkeypatch, cfg.batch)
    assert plan.info["fold"] == F and plan.info["fold_mode"] == 2
    plan.filter_transform(g.cuda())
    plan.forward(x.cuda())
    torch.cuda.synchronize()
    A, B, C = tc.synthesize(cfg.m, cfg.r, "0,1,-1,inf")
    _, st = wg.winograd_nd(x.numpy().astype(np.float64), g.numpy().astype(np.float64), cfg.padding, A, B, C)
    a, m, N = cfg.alpha, cfg.m, cfg.N
    T = cfg.tiles()
    S = st["Shat"].reshape((a ** (N - F),) + (a,) * F + (T, cfg.K))
    At = np.array([[float(v) for v in row] for row in A])          # m x alpha
    for f in range(F):                                             # contract the last F axes with A^T
        S = np.moveaxis(np.tensordot(At, S, axes=([1], [1 + f])), 0, 1 + f)
    Wref = S.reshape(a ** (N - F) * m ** F, T, cfg.K).transpose(0, 2, 1)      # [P/Q*MO][K][T]
    _, Mw = plan.workspace()
    Wg = Mw.cpu().double().numpy().reshape(-1)[: Wref.shape[0] * cfg.K * plan.info["T_stride"]]
    Wg = Wg.reshape(Wref.shape[0], cfg.K, plan.info["T_stride"])[:, :, :T]
    rel = np.linalg.norm(Wg - Wref) / np.linalg.norm(Wref)
    print("%s F=%d %s stage W relL2 %.3e" % (name, F, scheme, rel))
    assert rel <= tolerance(cfg)[0]
    plan.close()


def test_ufold_sizes(monkeypatch):
    # U' holds (P/Q) x (Q*C) x (MO*K) values: MO x the unfolded filter buffer
    cfg = UF_SMALL["c3"]
    sizes = {}
    for F in (0, 1):
        plan = _plan(cfg, F, "3xtf32", monkeypatch, 2)
        sizes[F] = (plan.info["K_stride"], pkg.wino_plan_sizes(plan.h)[1])
        assert plan.info["fold_mode"] == (2 if F else 0)
        plan.close()
    assert sizes[1][0] >= 2 * cfg.K
    # (P/Q) * (Q*C) = P*C rows of K_stride values, hi and lo buffers
    assert sizes[0][1] // sizes[0][0] == sizes[1][1] // sizes[1][0]


@pytest.mark.parametrize("name,F", [("c3", 2), ("c5", 2), ("c5", 3)])
def test_ufold_deeper_refused(name, F, monkeypatch):
    """F >= 2 is not planned: the Q*C-term TMEM accumulation chains exceed
    BASELINE.json's 2e-6 budget there (plan.cu kMaxUFoldF; measured 1.6e-6 to
    8.3e-6 relL2 on these ragged layers).  The plan falls back to no
    filter-side fold."""
    cfg = UF_SMALL[name]
    plan = _plan(cfg, F, "3xf16", monkeypatch, 2)
    assert plan.info["fold_mode"] != 2
    plan.close()


def test_ufold_default(monkeypatch):
    # default plans (no knobs): F(2^3, 3^3) takes the filter-side fold F = 1
    # on the 3xFP16 GEMM (measured fastest on c3); N = 4 keeps the epilogue
    # fold, F(4^N, 3^N) no fold
    for k in ("WINO_UFOLD", "WINO_FOLD", "WINO_GEMM_AUTO_MODE", "WINO_DFOLD"):
        monkeypatch.delenv(k, raising=False)
    # (c3: fold_mode 3 = the filter-side fold with the direct-axis fold on top)
    want = {"c3": (1, 3, 4), "c5": (2, 1, 3), "c2": (0, 0, 4), "c4": (0, 0, 4)}
    for name, (F, mode, gm) in want.items():
        cfg = CONFIGS[name]
        plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, 2, cfg.padding)
        got = (plan.info["fold"], plan.info["fold_mode"], plan.info["gemm_mode"])
        plan.close()
        assert got == (F, mode, gm), (name, got)
