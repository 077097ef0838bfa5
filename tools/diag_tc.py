"""Dev tool: dump the first tcgen05 GEMM stage (smem after conversion) and accumulator."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200 import wino
from paper_1611_06565_b200.workloads import SMALL, make_inputs
L = wino.lib()
p, n = ctypes.c_void_p(), ctypes.c_size_t()
L.wino_debug_tc_dump.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
assert L.wino_debug_tc_dump(ctypes.byref(p), ctypes.byref(n)) == 0
dbg = wino.device_view(p.value, (n.value // 4,))
cfg = SMALL["c1"]
x, g = make_inputs(cfg)
plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding)
plan.filter_transform(g.cuda()); y = plan.forward(x.cuda()); torch.cuda.synchronize()
info = plan.info; print(info)
V, M = plan.workspace()
d = dbg.cpu().numpy()
kc, bn = info["k_chunk"], info["n_blk"]
a_bytes = 128 * kc * 4; b_bytes = bn * kc * 4
A_hi = d[:a_bytes // 4]; A_lo = d[a_bytes // 4: 2 * a_bytes // 4]
B_hi = d[2 * a_bytes // 4: (2 * a_bytes + b_bytes) // 4]
print("A_hi nonzero", np.count_nonzero(A_hi), "A_lo nz", np.count_nonzero(A_lo), "B_hi nz", np.count_nonzero(B_hi))
Vt = V[0, :, :128].cpu().numpy()   # xi=0 [C][128]
print("V[0] c0 t0..8", Vt[0, :9])
print("A_hi first 40", A_hi[:40])
print("B_hi first 40", B_hi[:40])
U = plan.filter_tensor().cpu().numpy()
print("U_hi xi0 c0 k0..8", U[:8])
acc = d[65536:].reshape(128, 256)
print("acc nonzero", np.count_nonzero(acc), acc[:4, :6])
