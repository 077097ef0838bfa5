"""GPU parity of the 3xFP16 GEMM (gemm_f16.cu, WINO_GEMM_3XF16): V and U
scaled by powers of two and split into fp16 hi + lo on the kind::f16 tensor
path.  Against the float64 oracle at BASELINE.json's tolerances, on ragged
configs (every output) and the full c2 / c4 layers (sampled); and the
max|V| word is reset between forwards (a second forward on different data
gives that data's result)."""
import numpy as np
import pytest
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200 import wino
from paper_1611_06565_b200.workloads import CONFIGS, LayerConfig, make_inputs, tolerance
from oracle import direct, fp32model as fm

pytestmark = pytest.mark.gpu

F16 = wino.WINO_GEMM_3XF16
SMALLF = [
    LayerConfig("f16a", 3, 3, 40, 72, (6, 13, 10), 3, 1, 4, "relu_normal", "he"),    # c4-like, ragged
    LayerConfig("f16b", 2, 3, 64, 130, (29, 23), 3, 1, 4, "normal", "he"),           # K > 128: 2 n-blocks
    LayerConfig("f16c", 3, 2, 33, 96, (5, 13, 11), 3, 1, 2, "normal", "he"),         # F(2^3, 3^3), C odd
]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _plan(cfg, B=None):
    plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, B or cfg.batch, cfg.padding, gemm_mode=F16)
    assert plan.info["gemm_mode"] == F16
    return plan


@pytest.mark.parametrize("cfg", SMALLF, ids=lambda c: c.name)
def test_f16_every_output(cfg):
    x, g = make_inputs(cfg)
    plan = _plan(cfg)
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda()).cpu().double().numpy()
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
    rel, mx = fm.errors(y, ref)
    tl, tm = tolerance(cfg)
    print("%s 3xFP16 relL2=%.3e max=%.3e" % (cfg.name, rel, mx))
    assert rel <= tl and mx <= tm
    # a forward on other data (scaled x100: a different max|V|) gives that data's result
    x2 = x * 100.0
    y2 = plan.forward(x2.cuda()).cpu().double().numpy()
    rel2, _ = fm.errors(y2, ref * 100.0)
    assert rel2 <= tl
    plan.close()


@pytest.mark.parametrize("name", ["c4", "c2"])
def test_f16_full_size_sampled(name):
    cfg = CONFIGS[name]
    x, g = make_inputs(cfg)
    plan = _plan(cfg)
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda())
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    n = y.numel()
    idx = np.concatenate([np.arange(64), np.arange(n - 64, n), rng.integers(0, n, 4096)])
    ref = direct.direct_conv_at(x.numpy(), g.numpy(), cfg.pad, idx)
    got = y.reshape(-1)[torch.from_numpy(idx).cuda()].cpu().double().numpy()
    rel, mx = fm.errors(got, ref)
    tl, tm = tolerance(cfg)
    print("%s full 3xFP16 relL2=%.3e max=%.3e" % (name, rel, mx))
    assert rel <= tl and mx <= tm
    plan.close()


def test_f16_unsupported_shapes_are_errors():
    cfg = CONFIGS["c5"]                     # K = 32 <= 64
    with pytest.raises(pkg.WinoError) as ei:
        _plan(cfg, 1)
    assert ei.value.status == wino.WINO_ERR_UNSUPPORTED


def test_auto_scheme_choice():
    # WINO_GEMM_AUTO: 3xFP16 where measured faster (GEMM depth and width >= 128:
    # c2, c4, and c3 whose filter-side fold makes the GEMM 4 x 64 deep and
    # 2 x 128 wide), 3xTF32 elsewhere
    for name, want in (("c2", F16), ("c4", F16), ("c3", F16), ("c5", wino.WINO_GEMM_3XTF32)):
        cfg = CONFIGS[name]
        plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, 2, cfg.padding)
        assert plan.info["gemm_mode"] == want, (name, plan.info["gemm_mode"])
        plan.close()


def test_f16_host_path_and_filter_broadcast():
    # the host-buffer entry point (chunked forwards: max|V| cleared per chunk)
    # and a filter buffer copied into a second plan (the multi-GPU hook: the
    # scale travels with U) give the device path's bits
    cfg = SMALLF[1]
    x, g = make_inputs(cfg)
    p1 = _plan(cfg)
    p1.filter_transform(g.cuda())
    y = p1.forward(x.cuda()).cpu()
    yh = torch.empty_like(y).pin_memory()
    p1.forward_host(x.pin_memory(), yh)
    assert torch.equal(yh, y)
    p2 = _plan(cfg)
    p2.filter_tensor().copy_(p1.filter_tensor())
    p2.mark_ready()
    assert torch.equal(p2.forward(x.cuda()).cpu(), y)
    p1.close()
    p2.close()


# K = 200 (two n-blocks, the second ragged), C = 256 (four 64-channel chunks):
# the V-resident kernel (k_gemm_f16n) applies
F16N = LayerConfig("f16d", 3, 2, 256, 200, (4, 9, 10), 3, 1, 4, "relu_normal", "he")


@pytest.mark.parametrize("cfg", [F16N, SMALLF[1]], ids=lambda c: c.name)
def test_f16_vresident_bit_identical(cfg, monkeypatch):
    """k_gemm_f16n (V converted once per unit, kept in TMEM across the
    n-blocks) issues the same MMAs in the same order per output as
    k_gemm_f16p: bit-identical y; and within tolerance of the oracle."""
    x, g = make_inputs(cfg)
    ys = []
    for env in ("1", "0"):
        monkeypatch.setenv("WINO_F16N", env)
        plan = _plan(cfg)
        plan.filter_transform(g.cuda())
        ys.append(plan.forward(x.cuda()).cpu())
        plan.close()
    assert torch.equal(ys[0], ys[1])
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
    rel, mx = fm.errors(ys[0].double().numpy(), ref)
    tl, tm = tolerance(cfg)
    print("%s f16n relL2=%.3e max=%.3e" % (cfg.name, rel, mx))
    assert rel <= tl and mx <= tm
