"""Dev probe: one (config, GEMM variant) forward vs the FFMA GEMM; run each in
its own process under `timeout` (tools/variant_probe.sh)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, SMALL, make_inputs

name, var = sys.argv[1], sys.argv[2]
cfg = (SMALL if name.endswith("s") else CONFIGS)[name.rstrip("s")]
x, g = make_inputs(cfg)
os.environ["WINO_GEMM_VARIANT"] = var
plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding)
plan.filter_transform(g.cuda())
y = plan.forward(x.cuda())
torch.cuda.synchronize()
ref = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding, gemm_mode=1)
ref.filter_transform(g.cuda())
y1 = ref.forward(x.cuda())
torch.cuda.synchronize()
rel = ((y - y1).norm() / y1.norm()).item()
print(name, "variant", var, "->", plan.info["gemm_variant"], "bn", plan.info["n_blk"], "kc", plan.info["k_chunk"],
      "rel vs ffma %.2e" % rel, flush=True)
