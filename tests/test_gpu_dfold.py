"""GPU parity of the a5 direct-axis fold (fold_mode 3, xform_dfold.cu; DESIGN.md
reading #21): on top of the filter-side fold F = 1, B^T of the innermost axis
is folded into the cached filter as well, so the GEMM's A operand is Z (the
input transformed along the outer axes only, raw along the last axis) and the
innermost axis is computed directly:
  W[xo][o][k][t] = sum_{j,c} Z_xo[c][t_outer][m t_last + j] (g x_outer G)[xo][c][k][j - o]
(Eq. (4)-(5); the F(m, r) identity of PAPER.md:52-56
collapses sum_q A^T[o][q] B^T[q][j] G[q][i] to [i = j - o]).  Every output of
ragged layers against the float64 direct oracle at BASELINE.json's tolerance;
Z and W against the step-by-step float64 Winograd oracle; identical results
for batch shards; bias + ReLU; full-size c3 sampled."""
import numpy as np
import pytest
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, LayerConfig, make_inputs, tolerance
from oracle import direct, fp32model as fm, toomcook as tc, winograd as wg

pytestmark = pytest.mark.gpu

# F(2^3,3^3) layers the direct-axis fold takes (C a multiple of the k-chunk,
# 64 < K <= 128): ragged edge tiles on every axis, a slot count that is not a
# multiple of the 256-slot unit, K below the N tile, last-axis tile counts 1 .. 31
DF_CASES = {
    "d3a": LayerConfig("d3a", 3, 3, 64, 128, (5, 13, 11), 3, 1, 2, "normal", "he"),
    "d3b": LayerConfig("d3b", 3, 2, 32, 72, (4, 7, 61), 3, 1, 2, "normal", "he"),
    "d3c": LayerConfig("d3c", 3, 2, 64, 96, (6, 6, 2), 3, 1, 2, "normal", "he"),
    "d3d": LayerConfig("d3d", 3, 1, 32, 128, (3, 9, 20), 3, 0, 2, "normal", "he"),
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _plan(cfg, batch, monkeypatch, dfold=True):
    monkeypatch.setenv("WINO_DFOLD", "1" if dfold else "0")
    return pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, batch, cfg.padding)


@pytest.mark.parametrize("name", list(DF_CASES))
def test_dfold_every_output(name, monkeypatch):
    cfg = DF_CASES[name]
    x, g = make_inputs(cfg)
    plan = _plan(cfg, cfg.batch, monkeypatch)
    assert plan.info["fold"] == 1 and plan.info["fold_mode"] == 3, plan.info
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda()).cpu()
    plan.close()
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
    rel, mx = fm.errors(y.double().numpy(), ref)
    tl, tm = tolerance(cfg)
    print("%s dfold relL2=%.3e max=%.3e" % (cfg.name, rel, mx))
    assert rel <= tl and mx <= tm


def test_dfold_stage_z_and_w(monkeypatch):
    """Z (the GEMM's A operand, in the V workspace) against the float64 input
    transform of the two outer axes, and W (the GEMM's output) against the
    oracle's S_hat contracted with A^T along the last axis."""
    cfg = DF_CASES["d3a"]
    x, g = make_inputs(cfg)
    plan = _plan(cfg, cfg.batch, monkeypatch)
    assert plan.info["fold_mode"] == 3
    plan.filter_transform(g.cuda())
    plan.forward(x.cuda())
    torch.cuda.synchronize()
    A, B, C = tc.synthesize(cfg.m, cfg.r, "0,1,-1,inf")
    a, m = cfg.alpha, cfg.m
    Bt = np.array([[float(v) for v in row] for row in B])     # B^T as synthesised: alpha x alpha
    tiles = [-(-(d + 2 * cfg.pad - cfg.r + 1) // m) for d in cfg.dims]
    ext = [t * m + a - m for t in tiles]
    xp = np.zeros((cfg.batch, cfg.C) + tuple(ext))      # zero-padded input, index = input index + pad
    xn = x.numpy().astype(np.float64)
    p = cfg.pad
    xp[:, :, p:p + cfg.dims[0], p:p + cfg.dims[1], p:p + cfg.dims[2]] = xn
    # Zref[x0, x1, c, b, t0, t1, col] = sum_{i0,i1} B^T[x0][i0] B^T[x1][i1] xp[b, c, 2 t0 + i0, 2 t1 + i1, col]
    win0 = np.stack([xp[:, :, i0:i0 + m * tiles[0]:m] for i0 in range(a)], 0)           # [i0][b][c][t0][y][col]
    win = np.stack([win0[:, :, :, :, i1:i1 + m * tiles[1]:m] for i1 in range(a)], 1)    # [i0][i1][b][c][t0][t1][col]
    Zref = np.einsum("xi,yj,ijbctuv->xycbtuv", Bt, Bt, win)
    rows = cfg.batch * tiles[0] * tiles[1]
    S = 32                                          # slots per row of tiles (kernels.h kDfoldSlots)
    Tz = (rows * S + 255) // 256 * 256
    vptr, mptr = pkg.wino_workspace(plan.h)         # Z lives in the V region: [16 * 2][C][Tz]
    from paper_1611_06565_b200.wino import device_view
    Zg = device_view(vptr, (a * a * 2 * cfg.C * Tz,)).cpu().double().numpy().reshape(a, a, 2, cfg.C, Tz)
    tail = Zg[..., rows * S:]
    Zg = Zg[..., : rows * S].reshape(a, a, 2, cfg.C, cfg.batch, tiles[0], tiles[1], S)
    assert np.all(tail == 0)                        # the planes' tails stay zero
    for par in range(2):
        cols = Zref[..., par::2]                     # padded columns 2 i + par
        nc = cols.shape[-1]
        assert nc == tiles[2] + 1
        assert np.abs(Zg[:, :, par, ..., :nc] - cols).max() <= 4e-6 * np.abs(cols).max()
        assert np.all(Zg[:, :, par, ..., nc:] == 0)  # padding slots hold zeros
    # W as in tests/test_gpu_ufold.py
    _, st = wg.winograd_nd(xn, g.numpy().astype(np.float64), cfg.padding, A, B, C)
    T = cfg.tiles()
    S = st["Shat"].reshape((a * a, a, T, cfg.K))
    At = np.array([[float(v) for v in row] for row in A])
    S = np.moveaxis(np.tensordot(At, S, axes=([1], [1])), 0, 1)
    Wref = S.reshape(a * a * m, T, cfg.K).transpose(0, 2, 1)
    Ts = plan.info["T_stride"]
    Wg = device_view(mptr, (Wref.shape[0] * cfg.K * Ts,)).cpu().double().numpy().reshape(Wref.shape[0], cfg.K, Ts)[:, :, :T]
    rel = np.linalg.norm(Wg - Wref) / np.linalg.norm(Wref)
    print("dfold stage W relL2 %.3e" % rel)
    assert rel <= tolerance(cfg)[0]
    plan.close()


def test_dfold_close_to_ufold_and_batch_shards(monkeypatch):
    """Same layer through the plain filter-side fold (V path): both within the
    tolerance of each other; a forward of fewer samples than planned gives the
    same bits as the full batch (reading #8)."""
    cfg = DF_CASES["d3a"]
    x, g = make_inputs(cfg)
    pd = _plan(cfg, cfg.batch, monkeypatch, True)
    pd.filter_transform(g.cuda())
    yd = pd.forward(x.cuda()).cpu()
    y1 = pd.forward(x[:1].contiguous().cuda()).cpu()
    y2 = pd.forward(x.cuda()).cpu()
    pd.close()
    assert torch.equal(yd, y2)
    assert torch.equal(yd[:1], y1)
    pu = _plan(cfg, cfg.batch, monkeypatch, False)
    assert pu.info["fold_mode"] == 2
    pu.filter_transform(g.cuda())
    yu = pu.forward(x.cuda()).cpu()
    pu.close()
    rel, _ = fm.errors(yd.double().numpy(), yu.double().numpy())
    assert rel <= 2 * tolerance(cfg)[0]


def test_dfold_bias_relu(monkeypatch):
    cfg = DF_CASES["d3b"]
    x, g = make_inputs(cfg)
    b = torch.randn(cfg.K, generator=torch.Generator().manual_seed(5))
    plan = _plan(cfg, cfg.batch, monkeypatch)
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda()).cpu()
    yb = plan.forward(x.cuda(), bias=b.cuda(), relu=True).cpu()
    plan.close()
    assert torch.equal(yb, torch.clamp_min(y + b.view(1, cfg.K, 1, 1, 1), 0.0))


def test_dfold_not_taken_where_unsupported(monkeypatch):
    # more than 31 tiles along the last axis, or K outside (64, 128]: the plain filter-side fold / unfused plan
    for dims, C, K in (((4, 6, 64), 64, 128), ((4, 6, 10), 64, 64), ((4, 6, 10), 48, 128)):
        plan = pkg.Plan(3, dims, 2, 3, C, K, 2, (1, 1, 1))
        assert plan.info["fold_mode"] != 3, (dims, C, K, plan.info)
        plan.close()


def test_dfold_full_size_c3_sampled(monkeypatch):
    cfg = CONFIGS["c3"]
    x, g = make_inputs(cfg)
    plan = _plan(cfg, cfg.batch, monkeypatch)
    assert plan.info["fold_mode"] == 3, plan.info
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda()).cpu()
    plan.close()
    rng = np.random.default_rng(7)
    n = y.numel()
    idx = np.concatenate([np.arange(64), np.arange(n - 64, n), rng.integers(0, n, 4096)])
    ref = direct.direct_conv_at(x.numpy(), g.numpy(), cfg.pad, idx)
    rel, mx = fm.errors(y.reshape(-1)[torch.from_numpy(idx)].double().numpy(), ref)
    tl, tm = tolerance(cfg)
    print("c3 full dfold relL2=%.3e max=%.3e" % (rel, mx))
    assert rel <= tl and mx <= tm
