"""GPU parity on the large 3-D / 4-D layers the paper targets (C3D video,
PAPER.md:191; volumetric segmentation / connectomics and large volumes,
PAPER.md:40, 42, 145, 324): planes too large for one shared-memory slab of
the fused input transform are banded along axis 1 (info in_bands > 1), and
4-D layers with large planes likewise.  Full spatial sizes, small channel
counts (the oracle evaluates every sampled output by direct summation).
Tolerances: BASELINE.json's for F(2^N, 3^N) and F(4^N, 3^N) (north_star).
Each case also checks the banded plan against the generic multi-pass plan
(WINO_ND_GENERIC=1) within the same bound.
"""
import numpy as np
import pytest
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import LayerConfig, make_inputs, tolerance
from oracle import direct

pytestmark = pytest.mark.gpu

CASES = [
    # name, N, batch, C, K, dims, m, expect banded
    ("c3d_112_f2", 3, 2, 8, 16, (16, 112, 112), 2, True),
    ("c3d_112_f4", 3, 2, 8, 16, (16, 112, 112), 4, True),
    ("vol64_f2", 3, 1, 4, 8, (64, 64, 64), 2, False),
    ("vol128_f2", 3, 1, 4, 8, (128, 128, 128), 2, True),
    ("vol128_f4", 3, 1, 4, 8, (128, 128, 128), 4, True),
    ("4d_16x16x32x32", 4, 2, 4, 8, (16, 16, 32, 32), 2, True),
]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _sampled_check(cfg, x, g, y, seed=0):
    rng = np.random.default_rng(seed)
    n = y.numel()
    idx = np.concatenate([np.arange(64), np.arange(n - 64, n), rng.integers(0, n, 6000)])
    ref = direct.direct_conv_at(x.numpy(), g.numpy(), cfg.pad, idx)
    got = y.reshape(-1)[torch.from_numpy(idx)].double().numpy()
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    mx = float(np.abs(got - ref).max() / np.abs(ref).max())
    return rel, mx


@pytest.mark.parametrize("name,N,B,C,K,dims,m,banded", CASES)
def test_large_planes(name, N, B, C, K, dims, m, banded, monkeypatch):
    cfg = LayerConfig(name, N, B, C, K, dims, 3, 1, m, "normal", "he")
    x, g = make_inputs(cfg)
    tl, tm = tolerance(cfg)
    ys = {}
    for gen in ("0", "1"):
        monkeypatch.setenv("WINO_ND_GENERIC", gen)
        plan = pkg.Plan(N, dims, m, 3, C, K, B, cfg.padding)
        info = plan.info
        if gen == "0":
            assert info["axis_mode"] == 0                      # the fused kernels, not a refusal
            assert (info["in_bands"] > 1) == banded, info
        else:
            assert info["axis_mode"] == 2
        plan.filter_transform(g.cuda())
        y = plan.forward(x.cuda())
        torch.cuda.synchronize()
        ys[gen] = y.cpu()
        plan.close()
        rel, mx = _sampled_check(cfg, x, g, ys[gen])
        print("%s generic=%s bands=%d relL2=%.2e max=%.2e (tol %.0e/%.0e)" %
              (name, gen, info["in_bands"], rel, mx, tl, tm))
        assert rel <= tl and mx <= tm
    d = (ys["0"].double() - ys["1"].double()).norm() / ys["1"].double().norm()
    assert float(d) <= tl


def test_banded_equals_unbanded_bits(monkeypatch):
    # a plane that fits unbanded at the default thresholds, forced into bands
    # (dev knobs WINO_IN_BAND_KB / WINO_IN_TARGET_KB): the banded kernel
    # computes every V element by the same arithmetic, so y is bit-identical
    cfg = LayerConfig("band", 3, 2, 6, 10, (6, 40, 36), 3, 1, 4, "normal", "he")
    x, g = make_inputs(cfg)
    out = {}
    for kb in ("", "8"):
        if kb:
            monkeypatch.setenv("WINO_IN_BAND_KB", kb)       # band every slab over 8 KB ...
            monkeypatch.setenv("WINO_IN_TARGET_KB", "12")   # ... into bands near 12 KB
        plan = pkg.Plan(3, cfg.dims, 4, 3, cfg.C, cfg.K, 2, cfg.padding)
        out[kb] = (plan.info["in_bands"], None)
        plan.filter_transform(g.cuda())
        out[kb] = (plan.info["in_bands"], plan.forward(x.cuda()).cpu())
        plan.close()
    assert out[""][0] == 1 and out["8"][0] > 1
    assert torch.equal(out[""][1], out["8"][1])
