"""Dev probe: device time per forward of tiny layers (c1, and the paper's
Figure 4 at batch 1) replayed from a CUDA graph of 50 forwards (no host
overhead), tiny single-kernel path vs three kernels."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, make_inputs

for tiny in ("1", "0"):
    os.environ["WINO_TINY"] = tiny
    cfg = CONFIGS["c1"]
    x, g = make_inputs(cfg)
    p = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, 1, cfg.padding)
    p.filter_transform(g.cuda())
    xd = x.cuda()
    y = p.forward(xd)
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(50):
            p.forward(xd, y, s)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        gr.replay()
    b.record()
    torch.cuda.synchronize()
    print("c1 tiny=%s (plan tiny=%d): %.2f us per forward (graph replay)" % (tiny, p.info["tiny"],
                                                                          a.elapsed_time(b) / 20 / 50 * 1e3))
    p.close()
