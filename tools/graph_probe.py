"""Dev probe: eager vs CUDA-graph replay of plan.forward for fuse 0 / 4."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, make_inputs

torch.cuda.set_device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in sys.argv[1].split(","):
    cfg = CONFIGS[name]
    x, g = make_inputs(cfg)
    xd = x.cuda()
    for fuse in (0, 4):
        for mb in (["48"] if fuse == 0 else ["24", "48", "80"]):
            os.environ["WINO_CHUNK_MB"] = mb
            plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding, fuse=fuse)
            plan.filter_transform(g.cuda())
            y = torch.empty((cfg.batch, cfg.K) + cfg.out_dims, device="cuda")
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    plan.forward(xd, y, s.cuda_stream)
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                plan.forward(xd, y, s.cuda_stream)
            torch.cuda.synchronize()
            res = {}
            for mode in ("eager", "graph"):
                ts = []
                for i in range(20):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    with torch.cuda.stream(s):
                        a.record(s)
                        if mode == "eager":
                            plan.forward(xd, y, s.cuda_stream)
                        else:
                            gr.replay()
                        b.record(s)
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                ts.sort()
                res[mode] = ts[len(ts) // 2]
            print("%s fuse=%d chunkMB=%s chunk_slabs=%d eager=%.4f ms graph=%.4f ms" %
                  (name, fuse, mb, plan.info["chunk_slabs"], res["eager"], res["graph"]), flush=True)
            plan.close()
