"""Dev probe: wino_forward_host time vs pipeline chunk count (WINO_HOST_CHUNKS)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, make_inputs

for name in sys.argv[1].split(","):
    cfg = CONFIGS[name]
    x, g = make_inputs(cfg)
    plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding)
    plan.filter_transform(g.cuda())
    xh = x.pin_memory()
    yh = torch.empty((cfg.batch, cfg.K) + cfg.out_dims).pin_memory()
    s = torch.cuda.Stream()
    out = []
    for nch in [1, 2, 4, 6, 8, 12, 16]:
        os.environ["WINO_HOST_CHUNKS"] = str(nch)
        for _ in range(2):
            plan.forward_host(xh, yh, s.cuda_stream)
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            plan.forward_host(xh, yh, s.cuda_stream)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out.append("%d:%.3f" % (nch, sorted(ts)[2]))
    print(name, " ".join(out), flush=True)
    plan.close()
