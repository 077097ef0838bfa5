"""Stage-by-stage diagnostic (dev tool): U, V, M, y of the CUDA path vs the oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import SMALL, CONFIGS, make_inputs
from oracle import direct, toomcook as tc, winograd as wg

PTS = {4: "0,1,-1,inf", 6: "0,3/2,-3/2,2/3,-2/3,inf"}
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1"]
modes = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 3]
for name in names:
    cfg = SMALL[name]
    x, g = make_inputs(cfg)
    A, B, C = tc.synthesize(cfg.m, cfg.r, PTS[cfg.alpha])
    yref, st = wg.winograd_nd(x.numpy().astype(np.float64), g.numpy().astype(np.float64), cfg.padding, A, B, C)
    T = cfg.tiles()
    for mode in modes:
        plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding, gemm_mode=mode)
        info = plan.info
        plan.filter_transform(g.cuda())
        y = plan.forward(x.cuda()); torch.cuda.synchronize()
        P, Ts, Ks = info["n_points"], info["T_stride"], info["K_stride"]
        u = plan.filter_tensor().cpu().double().numpy()
        n = P * cfg.C * Ks
        U = (u[:n] + (u[n:2 * n] if mode != 1 else 0)).reshape(P, cfg.C, Ks)[:, :, :cfg.K]
        V, M = plan.workspace()
        Vg = V.cpu().double().numpy()[:, :, :T]; Mg = M.cpu().double().numpy()[:, :, :T]
        Vr = st["V"].transpose(0, 2, 1); Mr = st["Shat"].transpose(0, 2, 1); Ur = st["U"]
        rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
        print(name, "mode", mode, info)
        print("  U rel %.3e  V rel %.3e  M rel %.3e  y rel %.3e" % (rel(U, Ur), rel(Vg, Vr), rel(Mg, Mr), rel(y.cpu().double().numpy(), yref)))
        print("  |U| %.3e |V| %.3e |M| %.3e |y| %.3e" % (np.abs(U).max(), np.abs(Vg).max(), np.abs(Mg).max(), np.abs(y.cpu().numpy()).max()))
        if rel(Mg, Mr) > 1e-4:
            print("  M[0,:4,:6] gpu\n", Mg[0, :4, :6], "\n  ref\n", Mr[0, :4, :6])
        plan.close()
