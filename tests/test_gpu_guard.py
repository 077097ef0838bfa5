"""Memory-safety evidence without compute-sanitizer (closed on this pool,
profiles/r02_compute_sanitizer_refused.txt): every tensor the kernels touch
is a view into a larger allocation whose guard bands hold a canary value;
after filter transform and forward the guards must be intact (no stray
writes) and the outputs unchanged when the input's guards hold NaN (no
stray reads).  Every kernel family: fused 3xTF32 (each GEMM variant),
3xFP16, the folded GEMM (a5), the generic per-axis passes, banded slabs,
the host-buffer path."""
import numpy as np
import pytest
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import SMALL, LayerConfig, make_inputs

pytestmark = pytest.mark.gpu

GUARD = 4096          # floats on each side
CANARY = 1234.5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def guarded(shape, fill, inner=None):
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), fill, dtype=torch.float32, device="cuda")
    v = buf[GUARD:GUARD + n].view(shape)
    if inner is not None:
        v.copy_(inner)
    return buf, v


def guards_ok(buf, n, fill):
    g = torch.cat([buf[:GUARD], buf[GUARD + n:]])
    return bool(torch.all(g == fill)) if not np.isnan(fill) else bool(torch.all(torch.isnan(g)))


CASES = [
    ("c2", SMALL["c2"], None, {}),
    ("c4", SMALL["c4"], None, {}),
    ("c4_pair", SMALL["c4"], None, {"WINO_GEMM_VARIANT": "2"}),
    ("c4_ss", SMALL["c4"], None, {"WINO_GEMM_VARIANT": "0"}),
    ("c5", SMALL["c5"], None, {}),
    ("f16", LayerConfig("gf16", 3, 3, 40, 130, (6, 13, 10), 3, 1, 4, "relu_normal", "he"), 4, {}),
    ("fold", LayerConfig("gfold", 3, 2, 40, 48, (5, 13, 11), 3, 1, 2, "normal", "he"), None, {"WINO_FOLD": "2"}),
    ("generic", LayerConfig("ggen", 2, 2, 5, 7, (13, 11), 4, 1, 4, "normal", "he"), None, {}),
    ("banded", LayerConfig("gband", 3, 2, 6, 10, (6, 40, 36), 3, 1, 4, "normal", "he"), None,
     {"WINO_IN_BAND_KB": "8", "WINO_IN_TARGET_KB": "12"}),
]


@pytest.mark.parametrize("name,cfg,mode,env", CASES, ids=[c[0] for c in CASES])
def test_guard_bands(name, cfg, mode, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    x, g = make_inputs(cfg)
    plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding,
                    gemm_mode=mode or 0)
    # reference: plain contiguous tensors
    plan.filter_transform(g.cuda())
    y_ref = plan.forward(x.cuda()).clone()
    # guarded: NaN around x and g (reads past them would poison y), canary around y
    gb, gv = guarded(tuple(g.shape), float("nan"), g.cuda())
    xb, xv = guarded(tuple(x.shape), float("nan"), x.cuda())
    yb, yv = guarded(tuple(y_ref.shape), CANARY)
    plan.filter_transform(gv)
    plan.forward(xv, yv)
    torch.cuda.synchronize()
    assert guards_ok(yb, yv.numel(), CANARY), "%s: a kernel wrote outside y" % name
    assert guards_ok(xb, xv.numel(), float("nan")) and guards_ok(gb, gv.numel(), float("nan"))
    assert torch.equal(yv, y_ref), "%s: output depends on memory outside x / g" % name
    # host-buffer path into a guarded pinned buffer
    yh = torch.full((yv.numel() + 2 * GUARD,), CANARY, dtype=torch.float32).pin_memory()
    plan.forward_host(x.pin_memory(), yh[GUARD:GUARD + yv.numel()].view(tuple(y_ref.shape)))
    assert bool(torch.all(yh[:GUARD] == CANARY)) and bool(torch.all(yh[GUARD + yv.numel():] == CANARY))
    assert torch.equal(yh[GUARD:GUARD + yv.numel()].view(tuple(y_ref.shape)), y_ref.cpu())
    plan.close()
