"""Dev probe: per-stage times (instrumented pass) and roofline fractions of one
layer: python tools/stage_probe.py N dims m r C K B pad [env...]"""
import math
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.cost import stage_model

def layer(N, dims, m, r, C, K, B, pad):
    gen = torch.Generator("cpu").manual_seed(0)
    x = torch.randn((B, C) + tuple(dims), generator=gen).cuda()
    g = (torch.randn((K, C) + (r,) * N, generator=gen) * math.sqrt(2.0 / (C * r ** N))).cuda()
    p = pkg.Plan(N, dims, m, r, C, K, B, (pad,) * N)
    p.filter_transform(g)
    y = p.forward(x)
    for _ in range(3):
        p.forward(x, y)
    torch.cuda.synchronize()
    p.profile(True)
    for _ in range(5):
        p.forward(x, y)
    torch.cuda.synchronize()
    ms, calls = p.profile_read()
    st = stage_model(N, dims, m, r, C, K, B, (pad,) * N, hbm_gbs=6447, tf32_tflops=817)
    names = ["input_xform", "gemm", "output_xform"]
    print("N=%d dims=%s F(%d,%d) C=%d K=%d B=%d info=%s" % (N, dims, m, r, C, K, B,
          {k: p.info[k] for k in ("gemm_variant", "n_blk", "in_slab_tiles", "in_planes_per_cta")}))
    for n, v in zip(names, ms):
        t = v / calls
        print("  %-12s %.4f ms  roofline %.4f ms  frac %.2f" % (n, t, st[n]["roofline_ms"], st[n]["roofline_ms"] / t))
    p.close()

layer(2, (224, 224), 5, 4, 32, 32, 200, 0)
layer(2, (224, 224), 3, 4, 32, 32, 200, 0)
