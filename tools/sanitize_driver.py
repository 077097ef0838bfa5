"""Small forwards of every kernel family for compute-sanitizer (tools/sanitize.sh).
Each case runs one filter transform + one forward and checks the result against
the float64 oracle (so a silent corruption also fails)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_06565_b200 as pkg  # noqa: E402
from paper_1611_06565_b200.workloads import SMALL, LayerConfig, make_inputs, tolerance  # noqa: E402
from oracle import direct, fp32model as fm  # noqa: E402

torch.cuda.set_device(0)
which = sys.argv[1] if len(sys.argv) > 1 else "all"


def run(cfg, m=None, r=None, tol=None, label=""):
    x, g = make_inputs(cfg)
    plan = pkg.Plan(cfg.N, cfg.dims, m if m is not None else cfg.m, r if r is not None else cfg.r, cfg.C, cfg.K,
                    cfg.batch, cfg.padding)
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda()).cpu().double().numpy()
    torch.cuda.synchronize()
    info = plan.info
    plan.close()
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
    rel, mx = fm.errors(y, ref)
    tl, tm = tol if tol else tolerance(cfg)
    ok = rel <= tl and mx <= tm
    print("%-28s variant=%d axis_mode=%d bands=%d relL2=%.2e %s" % (label or cfg.name, info["gemm_variant"],
          info["axis_mode"], info["in_bands"], rel, "ok" if ok else "FAIL"), flush=True)
    return ok


ok = True
if which in ("all", "small"):
    for name in ("c1", "c2", "c3", "c4", "c5"):
        ok &= run(SMALL[name])
if which in ("all", "extra"):
    # banded slab (forced), generic fallback (alpha = 7), per-axis mixed plan
    os.environ["WINO_IN_BAND_KB"] = "8"
    os.environ["WINO_IN_TARGET_KB"] = "12"
    ok &= run(LayerConfig("band", 3, 2, 6, 10, (6, 40, 36), 3, 1, 4, "normal", "he"), label="banded F(4^3,3^3)")
    del os.environ["WINO_IN_BAND_KB"], os.environ["WINO_IN_TARGET_KB"]
    ok &= run(LayerConfig("a7", 2, 2, 5, 7, (13, 11), 4, 1, 4, "normal", "he"), tol=(1e-4, 1e-3),
              label="generic F(4,4)")
    cfg = LayerConfig("mix", 3, 2, 8, 12, (6, 13, 11), 3, 1, 2, "normal", "he")
    ok &= run(cfg, m=[2, 4, 4], r=[3, 3, 3], tol=(1e-5, 1e-4), label="mixed F(2x4x4,3^3)")
print("ALL_OK" if ok else "SOME_FAILED")
sys.exit(0 if ok else 1)
