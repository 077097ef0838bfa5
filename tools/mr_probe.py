"""Dev probe: GPU relL2 / max error vs the float64 oracle for the run-time
table instantiations (arbitrary (m, r), SPEC-order points)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import LayerConfig, make_inputs
from oracle import direct

torch.cuda.set_device(0)
shapes = {1: (37,), 2: (13, 11), 3: (6, 7, 9)}
for (m, r) in [(3, 2), (2, 3), (3, 3), (3, 4), (4, 3), (3, 6), (4, 5), (5, 4)]:
    for N in (1, 2, 3):
        if (m + r - 1) > 6 and N == 3:
            pass
        cfg = LayerConfig("mr", N, 2, 5, 7, shapes[N], r, 1, m, "normal", "he")
        x, g = make_inputs(cfg)
        for mode in (0, 1):
            try:
                plan = pkg.Plan(N, cfg.dims, m, r, 5, 7, 2, cfg.padding, gemm_mode=mode, points=None)
            except Exception as e:
                print("m=%d r=%d N=%d: %s" % (m, r, N, e))
                break
            plan.filter_transform(g.cuda())
            y = plan.forward(x.cuda()).cpu().double().numpy()
            ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
            rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
            mx = np.abs(y - ref).max() / np.abs(ref).max()
            print("m=%d r=%d N=%d mode=%d alpha=%d relL2=%.2e max=%.2e" % (m, r, N, mode, m + r - 1, rel, mx),
                  flush=True)
            plan.close()
