"""Dev tool: a few forwards of one per-axis bench workload (for ncu captures):
python tools/run_nd.py c3t [reps]"""
import math
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1611_06565_b200 as pkg

w = bench.ND_WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c3t"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
gen = torch.Generator("cpu").manual_seed(0)
x = torch.randn((w["B"], w["C"]) + w["dims"], generator=gen).cuda()
g = torch.randn((w["K"], w["C"]) + w["r"], generator=gen).cuda() * math.sqrt(2.0 / (w["C"] * math.prod(w["r"])))
plan = pkg.Plan(w["N"], w["dims"], list(w["m"]), list(w["r"]), w["C"], w["K"], w["B"], w["pad"])
plan.filter_transform(g)
for _ in range(reps):
    y = plan.forward(x)
torch.cuda.synchronize()
print("ok", plan.info["axis_mode"], plan.info["gemm_variant"], tuple(y.shape))
