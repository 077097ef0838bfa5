"""GPU parity of the a5 epilogue fusion (gemm_fold.cu + xform_fold.cu): the
output transform of the F innermost axes applied in the GEMM epilogue, the
rest in a4.  Every output of shrunken and
ragged configs against the float64 direct oracle at BASELINE.json's
tolerances, and against the unfused plan; full-size configs sampled."""
import numpy as np
import pytest
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, SMALL, LayerConfig, make_inputs, tolerance
from oracle import direct, fp32model as fm, toomcook as tc, winograd as wg

pytestmark = pytest.mark.gpu

CASES = [("c3", 1), ("c3", 2), ("c5", 2), ("c2", 1)]
# ragged shapes the folded kernels accept (k-chunk 32: C >= 32): partial last
# channel chunk, K not a multiple of the N tile, partial edge tiles, T not a
# multiple of 128
FOLD_SMALL = {
    "c3": LayerConfig("f3s", 3, 2, 40, 48, (5, 13, 11), 3, 1, 2, "normal", "he"),
    "c5": LayerConfig("f5s", 4, 2, 36, 20, (3, 4, 5, 6), 3, 1, 2, "normal", "he"),
    "c2": LayerConfig("f2s", 2, 2, 32, 40, (29, 23), 3, 1, 4, "normal", "he"),
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _run(cfg, F, monkeypatch, x, g, bias=None, relu=False):
    monkeypatch.setenv("WINO_FOLD", str(F))
    plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, x.shape[0], cfg.padding)
    info = plan.info
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda(), bias=bias, relu=relu).cpu()
    plan.close()
    return y, info


@pytest.mark.parametrize("name,F", CASES)
def test_fold_small_every_output(name, F, monkeypatch):
    cfg = FOLD_SMALL[name]
    x, g = make_inputs(cfg)
    y, info = _run(cfg, F, monkeypatch, x, g)
    assert info["fold"] == F, info
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
    rel, mx = fm.errors(y.double().numpy(), ref)
    tl, tm = tolerance(cfg)
    print("%s fold F=%d relL2=%.3e max=%.3e" % (cfg.name, F, rel, mx))
    assert rel <= tl and mx <= tm
    y0, info0 = _run(cfg, 0, monkeypatch, x, g)
    assert info0["fold"] == 0
    assert fm.errors(y.double().numpy(), y0.double().numpy())[0] <= tl


@pytest.mark.parametrize("name,F", [("c3", 1), ("c5", 2)])
def test_fold_bias_relu(name, F, monkeypatch):
    cfg = FOLD_SMALL[name]
    x, g = make_inputs(cfg)
    b = torch.randn(cfg.K, generator=torch.Generator().manual_seed(5))
    y, _ = _run(cfg, F, monkeypatch, x, g)
    yb, _ = _run(cfg, F, monkeypatch, x, g, bias=b.cuda(), relu=True)
    shape = (1, cfg.K) + (1,) * cfg.N
    assert torch.equal(yb, torch.clamp_min(y + b.view(shape), 0.0))


@pytest.mark.parametrize("name,F", [("c3", 1), ("c3", 2), ("c5", 2)])
def test_fold_full_size_sampled(name, F, monkeypatch):
    cfg = CONFIGS[name]
    x, g = make_inputs(cfg)
    y, info = _run(cfg, F, monkeypatch, x, g)
    assert info["fold"] == F
    rng = np.random.default_rng(7)
    n = y.numel()
    idx = np.concatenate([np.arange(64), np.arange(n - 64, n), rng.integers(0, n, 4096)])
    ref = direct.direct_conv_at(x.numpy(), g.numpy(), cfg.pad, idx)
    rel, mx = fm.errors(y.reshape(-1)[torch.from_numpy(idx)].double().numpy(), ref)
    tl, tm = tolerance(cfg)
    print("%s full fold F=%d relL2=%.3e max=%.3e" % (name, F, rel, mx))
    assert rel <= tl and mx <= tm


def test_fold_ragged_k_and_tiles(monkeypatch):
    # K not a multiple of the fold kernel's N tile, T not a multiple of 128
    cfg = LayerConfig("fr", 3, 3, 36, 70, (5, 9, 7), 3, 1, 2, "normal", "he")
    x, g = make_inputs(cfg)
    y, info = _run(cfg, 1, monkeypatch, x, g)
    assert info["fold"] == 1
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), 1)
    rel, mx = fm.errors(y.double().numpy(), ref)
    assert rel <= 2e-6 and mx <= 1e-4


@pytest.mark.parametrize("name,F", [("c3", 1), ("c3", 2), ("c5", 2)])
def test_fold_stage_w(name, F, monkeypatch):
    """W (the folded GEMM's output, in the M workspace) against the oracle:
    S_hat of Eq. (5) with A^T applied along the last F axes (Eq. (4))."""
    cfg = FOLD_SMALL[name]
    x, g = make_inputs(cfg)
    monkeypatch.setenv("WINO_FOLD", str(F))
    plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding)
    assert plan.info["fold"] == F
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
    print("%s F=%d stage W relL2 %.3e" % (name, F, rel))
    assert rel <= tolerance(cfg)[0]
    plan.close()


def test_fold_off_where_infeasible_or_slower(monkeypatch):
    # default plans: the epilogue fold F = 2 for F(2^4, 3^4) (measured
    # faster); F(2^3, 3^3) takes the filter-side fold F = 1 instead
    # (tests/test_gpu_ufold.py); no fold for F(4^N, 3^N), for small channel
    # counts (k-chunk < 32) or chunked plans
    monkeypatch.delenv("WINO_FOLD", raising=False)
    monkeypatch.delenv("WINO_UFOLD", raising=False)
    monkeypatch.delenv("WINO_DFOLD", raising=False)
    # (c3: the filter-side fold with the direct-axis fold on top, fold_mode 3, tests/test_gpu_dfold.py)
    for name, want in (("c3", (1, 3)), ("c5", (2, 1)), ("c2", (0, 0)), ("c4", (0, 0))):
        cfg = CONFIGS[name]
        plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, 2, cfg.padding)
        assert (plan.info["fold"], plan.info["fold_mode"]) == want, (name, plan.info)
        plan.close()
    cfg = SMALL["c3"]                                   # C = 16: k-chunk 16
    plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, 2, cfg.padding)
    assert plan.info["fold"] == 0
    plan.close()
