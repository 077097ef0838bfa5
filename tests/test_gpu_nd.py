"""GPU parity for per-axis transforms F(m_1 x .. x m_N, r_1 x .. x r_N)
(the fused distinct-axis-0 kernels for F(2,3) x F(4,3)^2 and F(4,3) x F(2,3)^2,
the generic multi-pass path for every other mix)
(Eq. (4) indexes B_n, A_n, C_n by axis):
wino_plan_create_nd against the float64 direct oracle on ragged shapes with
padding, both GEMM schemes; e.g. F(2,3) along time with F(4,3) along space
(the C3D-style video layer), anisotropic kernels such as 2x3 and 1x3.

Tolerance (reading #17): from the arithmetic, not the device --
oracle.fp32model's float32 / 3xTF32 model of Eq. (4)-(5) with the same
per-axis transforms on the same inputs; the GPU must stay within K_REL = 4x
its relL2 and K_MAX = 8x its max-abs / max|y|.
"""
import math

import numpy as np
import pytest
import torch

import paper_1611_06565_b200 as pkg
from oracle import direct, fp32model as fm

pytestmark = pytest.mark.gpu

CASES = [
    # N, dims, m per axis, r per axis, pad, B, C, K
    (3, (8, 14, 13), (2, 4, 4), (3, 3, 3), (1, 1, 1), 2, 16, 24),   # time F(2,3) x space F(4,3)
    (3, (7, 9, 10), (4, 2, 2), (3, 3, 3), (1, 1, 1), 2, 8, 12),
    (2, (17, 13), (4, 2), (3, 3), (1, 1), 3, 12, 20),
    (2, (15, 19), (3, 2), (2, 3), (0, 1), 2, 10, 9),                  # anisotropic 2x3 kernel
    (2, (9, 23), (2, 4), (1, 3), (0, 1), 2, 8, 8),                    # 1x3 kernel
    (3, (6, 11, 12), (1, 4, 4), (1, 3, 3), (0, 1, 1), 2, 8, 16),      # 1x3x3 (2-D kernels in a 3-D net)
    (4, (4, 5, 6, 7), (2, 2, 3, 2), (3, 2, 2, 3), (1, 0, 0, 1), 2, 4, 6),
    (1, (40,), (5,), (4,), (2,), 2, 6, 7),                            # N = 1 (uniform: fused path)
    (3, (6, 13, 12), (2, 1, 1), (3, 1, 1), (1, 0, 0), 2, 8, 8),      # 3x1x1 temporal kernel
    (3, (5, 12, 16), (1, 2, 2), (1, 3, 3), (0, 1, 1), 2, 8, 8),      # 1x3x3 with F(2,3) spatial
    (2, (14, 12), (4, 1), (3, 1), (1, 0), 2, 8, 8),                   # 3x1
]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _inputs(dims, r, B, C, K, seed=0):
    gen = torch.Generator("cpu").manual_seed(seed)
    x = torch.randn((B, C) + tuple(dims), generator=gen)
    g = torch.randn((K, C) + tuple(r), generator=gen) * math.sqrt(2.0 / (C * math.prod(r)))
    return x.contiguous(), g.contiguous()


def _tol(x, g, pad, m, r, ref):
    """(tol_rel, tol_max) from the float32 model on these inputs."""
    tl, tm, mrel, mmax = fm.model_tolerance(x, g, pad, tuple(m), tuple(r), ref)
    return tl, tm


@pytest.mark.parametrize("gemm_mode", [0, 1])
@pytest.mark.parametrize("N,dims,m,r,pad,B,C,K", CASES)
def test_per_axis_parity(N, dims, m, r, pad, B, C, K, gemm_mode):
    x, g = _inputs(dims, r, B, C, K)
    plan = pkg.Plan(N, dims, list(m), list(r), C, K, B, pad, gemm_mode=gemm_mode)
    assert plan.info["n_points"] == math.prod(a + b - 1 for a, b in zip(m, r))
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda()).cpu().double().numpy()
    plan.close()
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), pad)
    assert y.shape == ref.shape
    rel, mx = fm.errors(y, ref)
    tl, tm = _tol(x.numpy(), g.numpy(), pad, m, r, ref)
    print("m=%s r=%s mode=%d relL2=%.2e max=%.2e tol=%.1e/%.1e" % (m, r, gemm_mode, rel, mx, tl, tm))
    assert rel <= tl and mx <= tm


@pytest.mark.parametrize("N,dims,m,r,pad,B,C,K", [CASES[0], CASES[1], CASES[2], CASES[5], CASES[8], CASES[9],
                                                   CASES[10],
                                                   (2, (21, 30), (2, 4), (3, 3), (1, 1), 3, 12, 20),
                                                   (3, (9, 30, 29), (2, 4, 4), (3, 3, 3), (1, 1, 1), 3, 20, 40)])
def test_fused_mixed_axis0_equals_generic(N, dims, m, r, pad, B, C, K, monkeypatch):
    # a distinct axis-0 F(m0, 3) over F(m, 3) on the other axes runs the fused
    # kernels (xform_mixed.cu); the generic multi-pass path computes the same
    # transforms with another summation order: both within tolerance, close
    x, g = _inputs(dims, r, B, C, K, seed=5)
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), pad)
    ys = []
    for generic in ("0", "1"):
        monkeypatch.setenv("WINO_ND_GENERIC", generic)
        plan = pkg.Plan(N, dims, list(m), list(r), C, K, B, pad)
        assert plan.info["axis_mode"] == (2 if generic == "1" else 1)
        plan.filter_transform(g.cuda())
        ys.append(plan.forward(x.cuda()).cpu().double().numpy())
        plan.close()
    tol, tmax = _tol(x.numpy(), g.numpy(), pad, m, r, ref)
    for y in ys:
        rel, mx = fm.errors(y, ref)
        assert rel <= tol and mx <= tmax, (rel, mx)
    assert np.linalg.norm(ys[0] - ys[1]) / np.linalg.norm(ref) <= tol


def test_per_axis_bias_relu_and_host_path():
    N, dims, m, r, pad, B, C, K = CASES[0]
    x, g = _inputs(dims, r, B, C, K, seed=3)
    bias = torch.randn(K, generator=torch.Generator().manual_seed(9))
    plan = pkg.Plan(N, dims, list(m), list(r), C, K, B, pad)
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda()).cpu()
    yb = plan.forward(x.cuda(), bias=bias.cuda(), relu=True).cpu()
    # Eq. (2) epilogue: f(b + conv), in the spatial domain after A^T
    assert torch.equal(yb, torch.clamp_min(y + bias.view(1, K, 1, 1, 1), 0.0))
    # host-buffer entry point = device entry point, bit for bit
    yh = torch.empty_like(y).pin_memory()
    plan.forward_host(x.pin_memory(), yh)
    assert torch.equal(yh, y)
    plan.close()


def test_equal_axes_take_the_fused_plan():
    # per-axis entry point with equal (m_n, r_n): the single-(m, r) plan, same bits
    x, g = _inputs((13, 11), (3, 3), 2, 8, 8)
    p1 = pkg.Plan(2, (13, 11), [4, 4], [3, 3], 8, 8, 2, (1, 1))
    p2 = pkg.Plan(2, (13, 11), 4, 3, 8, 8, 2, (1, 1))
    assert p1.info["axis_mode"] == p2.info["axis_mode"] == 0
    for p in (p1, p2):
        p.filter_transform(g.cuda())
    assert torch.equal(p1.forward(x.cuda()), p2.forward(x.cuda()))
    p1.close()
    p2.close()


def test_per_axis_errors():
    with pytest.raises(pkg.WinoError):                 # alpha_0 = 9 > 8
        pkg.Plan(2, (16, 16), [6, 2], [4, 3], 4, 4, 1, (1, 1))
    with pytest.raises(ValueError):                    # points / fusion not per axis
        pkg.Plan(2, (16, 16), [2, 4], [3, 3], 4, 4, 1, (1, 1), fuse=4)


@pytest.mark.parametrize("name", ["c3t", "c3s133", "c3t311"])
def test_bench_per_axis_workloads_full_size_sampled(name):
    # the bench's per-axis workloads at full size, in the bench's launch
    # configuration: 4096 random outputs plus the first / last 64, each
    # computed one by one by the float64 oracle
    import bench
    w = bench.ND_WORKLOADS[name]
    gen = torch.Generator("cpu").manual_seed(0)
    x = torch.randn((w["B"], w["C"]) + w["dims"], generator=gen)
    g = torch.randn((w["K"], w["C"]) + w["r"], generator=gen) * math.sqrt(2.0 / (w["C"] * math.prod(w["r"])))
    plan = pkg.Plan(w["N"], w["dims"], list(w["m"]), list(w["r"]), w["C"], w["K"], w["B"], w["pad"])
    assert plan.info["axis_mode"] == 1
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda()).cpu().double().numpy()
    plan.close()
    rng = np.random.default_rng(2)
    idx = np.concatenate([np.arange(64), np.arange(y.size - 64, y.size), rng.integers(0, y.size, 4096)])
    ref = direct.direct_conv_at(x.numpy(), g.numpy(), w["pad"], idx)
    got = y.reshape(-1)[idx]
    rel, mx = fm.errors(got, ref)
    # model bound on a batch-1 slice of the same inputs (the error statistics
    # of a sample are those of the batch)
    xs, gs = x[:1].numpy(), g.numpy()
    ref1 = direct.direct_conv_f64(xs, gs, w["pad"])
    tl, tm = _tol(xs, gs, w["pad"], w["m"], w["r"], ref1)
    print("%s sampled relL2=%.2e max=%.2e tol=%.1e/%.1e" % (name, rel, mx, tl, tm))
    assert rel <= tl and mx <= tm
