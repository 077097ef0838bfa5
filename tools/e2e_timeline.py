"""Dev probe: timeline of a host-buffer pipeline built from the public device
API (H2D on one stream, forward on another, D2H on a third) with events after
every chunk's copy / forward / copy -- shows where wino_forward_host's time goes."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import CONFIGS, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = CONFIGS[name]
x, g = make_inputs(cfg)
B = cfg.batch
plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, B, cfg.padding)
plan.filter_transform(g.cuda())
xh = x.pin_memory()
yh = torch.empty((B, cfg.K) + cfg.out_dims).pin_memory()
xd = torch.empty_like(x, device="cuda")
yd = torch.empty(yh.shape, device="cuda")
s_in, s_fw, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
# forward time per chunk size (device resident)
for nb in [1, 2, 4, 8, 16, 32]:
    for _ in range(3):
        plan.forward(xd[:nb], yd[:nb], s_fw)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s_fw)
    for _ in range(10):
        plan.forward(xd[:nb], yd[:nb], s_fw)
    b.record(s_fw)
    torch.cuda.synchronize()
    print("forward B=%d: %.4f ms" % (nb, a.elapsed_time(b) / 10))


def ev():
    return torch.cuda.Event(enable_timing=True)


for nch in [8, 16]:
    for rep in range(3):
        t0 = ev()
        t0.record(s_in)
        s_out.wait_stream(s_in)
        last = None
        for i in range(nch):
            b0, b1 = B * i // nch, B * (i + 1) // nch
            with torch.cuda.stream(s_in):
                xd[b0:b1].copy_(xh[b0:b1], non_blocking=True)
                e1 = ev(); e1.record(s_in)
            s_out.wait_event(e1)
            with torch.cuda.stream(s_out):
                yh[b0:b1].copy_(yd[b0:b1], non_blocking=True)
                last = ev(); last.record(s_out)
        torch.cuda.synchronize()
    print("copies only nch=%d total %.3f ms" % (nch, t0.elapsed_time(last)))

for nch in [4, 8, 16]:
    for rep in range(3):
        t0 = ev()
        t0.record(s_in)
        s_fw.wait_stream(s_in)
        s_out.wait_stream(s_in)
        marks = []
        for i in range(nch):
            b0, b1 = B * i // nch, B * (i + 1) // nch
            with torch.cuda.stream(s_in):
                xd[b0:b1].copy_(xh[b0:b1], non_blocking=True)
                e1 = ev(); e1.record(s_in)
            s_fw.wait_event(e1)
            plan.forward(xd[b0:b1], yd[b0:b1], s_fw)
            e2 = ev(); e2.record(s_fw)
            s_out.wait_event(e2)
            with torch.cuda.stream(s_out):
                yh[b0:b1].copy_(yd[b0:b1], non_blocking=True)
                e3 = ev(); e3.record(s_out)
            marks.append((e1, e2, e3))
        torch.cuda.synchronize()
    print("nch=%d total %.3f ms" % (nch, t0.elapsed_time(marks[-1][2])))
    for i, (e1, e2, e3) in enumerate(marks):
        print("  chunk %2d  h2d_done %.3f  fw_done %.3f  d2h_done %.3f" %
              (i, t0.elapsed_time(e1), t0.elapsed_time(e2), t0.elapsed_time(e3)))
