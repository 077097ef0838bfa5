"""Dev probe: CTA-pair GEMM vs single-CTA GEMM on shrunken + full configs."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, SMALL, make_inputs

torch.cuda.set_device(0)
for name in sys.argv[1].split(","):
    cfg = (SMALL if name.endswith("s") else CONFIGS)[name.rstrip("s")]
    x, g = make_inputs(cfg)
    ys = []
    for var in ("2", "1"):
        os.environ["WINO_GEMM_VARIANT"] = var
        plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding)
        plan.filter_transform(g.cuda())
        y = plan.forward(x.cuda())
        torch.cuda.synchronize()
        ys.append(y.cpu())
        plan.close()
    d = (ys[0] - ys[1]).abs().max().item()
    print(name, "max|pair - single| =", d, "equal:", torch.equal(ys[0], ys[1]), flush=True)
