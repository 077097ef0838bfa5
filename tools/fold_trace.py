"""Run one folded forward with WINO_FOLD_TRACE and print CTA 0's pipeline
event latencies (dev probe of gemm_fold.cu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_06565_b200 as pkg  # noqa: E402
from paper_1611_06565_b200.workloads import CONFIGS, make_inputs  # noqa: E402

name = sys.argv[1]
cfg = CONFIGS[name]
x, g = make_inputs(cfg)
plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding)
plan.filter_transform(g.cuda())
xd = x.cuda()
path = os.environ["WINO_FOLD_TRACE"]
for _ in range(3):
    plan.forward(xd)
torch.cuda.synchronize()
t = np.fromfile(path, dtype=np.uint64).astype(np.int64).reshape(5, 4, 256)
names = {(0, 0): "Vp issue", (4, 0): "Up issue(g)", (1, 1): "cv aempty(g)", (1, 2): "cv done(g)",
         (2, 0): "mma waited(g)", (2, 2): "mma issued(g)", (3, 0): "epi tfull(g)", (3, 1): "epi done(g)"}
t0 = min(v for v in t[t > 0].ravel())
n = 24
for (r, e), nm in names.items():
    row = t[r, e, :n]
    print("%-14s" % nm, " ".join("%6d" % ((v - t0) if v else -1) for v in row))
def per(r, e):
    v = t[r, e]
    idx = np.nonzero(v)[0]
    idx = idx[(idx >= 20) & (idx < 200)]
    return np.diff(v[idx]).mean() if len(idx) > 2 else float("nan")
print("period cycles: conv/g %.0f  mma/g %.0f  Vp/chunk %.0f  Up/g %.0f  epi/g %.0f" % (per(1, 2), per(2, 2), per(0, 0), per(4, 0), per(3, 1)))
w = t[2, 0, 20:200]; i = t[2, 2, 20:200]
print("mma: waited->issued median %d, issued->next waited median %d" % (np.median(i - w), np.median(t[2, 0, 21:201] - i)))
