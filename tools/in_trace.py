"""Dev probe: per-CTA timeline of the a2 input transform (WINO_IN_TRACE).

Runs a config's forward a few times, then one traced forward; the library
writes one line per CTA (SM, %globaltimer at start / slabs landed / axis-0
pass done / end, ns).  Prints per-phase statistics and the SM occupancy
over time.  Usage: python tools/in_trace.py c4 [out.txt]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
path = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/in_trace_%s.txt" % name
cfg = CONFIGS[name]
x, g = make_inputs(cfg)
plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding, device=0)
plan.filter_transform(g.cuda())
xd = x.cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    plan.forward(xd)
torch.cuda.synchronize()
for rep in range(2):
    flush.fill_(rep)
    flush.sum()
    torch.cuda.synchronize()
    os.environ["WINO_IN_TRACE"] = path
    plan.forward(xd)
    torch.cuda.synchronize()
    del os.environ["WINO_IN_TRACE"]
d = np.loadtxt(path, dtype=np.int64)
sm, t0, tl, tp, te = d[:, 0], d[:, 1], d[:, 2], d[:, 3], d[:, 4]
base = t0.min()
print(name, "CTAs", len(d), "info", plan.info)
print("kernel span %.1f us (first start -> last end)" % ((te.max() - base) / 1e3))
ok = tl > 0
q = lambda a: "p10 %.2f p50 %.2f p90 %.2f mean %.2f" % tuple(np.percentile(a, [10, 50, 90]).tolist() + [a.mean()])
print("load  (start->landed) us:", q((tl[ok] - t0[ok]) / 1e3))
print("phase1(landed->pass)  us:", q((tp[ok] - tl[ok]) / 1e3))
print("phase2(pass->end)     us:", q((te[ok] - tp[ok]) / 1e3))
print("life  (start->end)    us:", q((te - t0) / 1e3))
# per SM: gaps between a CTA's end and the next CTA start in the same slot
gaps = []
conc = []
for s in np.unique(sm):
    idx = np.where(sm == s)[0]
    st = np.sort(t0[idx]); en = np.sort(te[idx])
    # concurrency sampled at every start
    for t in st:
        conc.append(int(((t0[idx] <= t) & (te[idx] > t)).sum()))
print("CTAs per SM: %s" % np.bincount(np.bincount(sm)).nonzero()[0].tolist())
print("concurrent CTAs on the SM at each CTA start: mean %.2f" % np.mean(conc))
# SM-occupancy timeline (fraction of CTA slots busy, 10 bins)
span = te.max() - base
bins = np.linspace(0, span, 11)
busy = []
for i in range(10):
    a, b = base + bins[i], base + bins[i + 1]
    ov = np.clip(np.minimum(te, b) - np.maximum(t0, a), 0, None).sum()
    busy.append(ov / (b - a) / len(np.unique(sm)))
print("mean CTAs resident per SM per tenth of the kernel:", " ".join("%.2f" % v for v in busy))
# phase mix over time: how many CTAs are loading / in phase 1 / in phase 2
for i in range(10):
    a, b = base + bins[i], base + bins[i + 1]
    f = lambda s0, s1: np.clip(np.minimum(s1, b) - np.maximum(s0, a), 0, None).sum() / (b - a) / len(np.unique(sm))
    print("  tenth %d: load %.2f phase1 %.2f phase2 %.2f" % (i, f(t0, tl), f(tl, tp), f(tp, te)))
