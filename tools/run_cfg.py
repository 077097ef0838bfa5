"""Dev tool: run one config's forward on cuda:0 stage by stage and report
errors / per-stage parity (python tools/run_cfg.py c2 [small])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, SMALL, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = (SMALL if "small" in sys.argv else CONFIGS)[name]
x, g = make_inputs(cfg)
plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding)
print("plan", plan.info, flush=True)
plan.filter_transform(g.cuda())
torch.cuda.synchronize()
print("filter ok", flush=True)
y = plan.forward(x.cuda())
torch.cuda.synchronize()
print("forward ok", float(y.abs().max()), flush=True)
