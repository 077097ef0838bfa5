"""Dev probe: Figure 4 chain at batch 1 / 20: eager forwards vs CUDA-graph replay."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import NETS, make_net_inputs

for name in ("fig4_f54", "fig4_f34"):
    for B in (1, 20):
        cfg = NETS[name]
        x, gs = make_net_inputs(cfg, batch=B)
        layers = [(l.N, l.dims, l.m, l.r, l.C, l.K, l.padding) for l in cfg.layers]
        net = pkg.Net(layers, B)
        net.filter_transform([g.cuda() for g in gs])
        xd = x.cuda()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                net.forward(xd, s)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(50):
            net.forward(xd, s)
        b.record(s)
        torch.cuda.synchronize()
        eager = a.elapsed_time(b) / 50
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            net.forward(xd, s)
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        a.record()
        for _ in range(50):
            gr.replay()
        b.record()
        torch.cuda.synchronize()
        print("%s B=%d eager %.4f ms  graph %.4f ms" % (name, B, eager, a.elapsed_time(b) / 50))
        net.close()
