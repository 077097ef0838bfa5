"""Dev probe: chunked H2D/D2H copy pipelines (no kernels), 51 MB each way
(c2's x and y): uniform chunks on one stream per direction vs chunks spread
round-robin over several streams per direction."""
import torch

n = 51380224 // 4
xh = torch.empty(n).pin_memory(); yh = torch.empty(n).pin_memory()
xd = torch.empty(n, device="cuda"); yd = torch.empty(n, device="cuda")


def ev():
    return torch.cuda.Event(enable_timing=True)


def run(nch, nstr):
    s_in = [torch.cuda.Stream() for _ in range(nstr)]
    s_out = [torch.cuda.Stream() for _ in range(nstr)]
    best = 1e9
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = ev(); t0.record()
        for s in s_in + s_out:
            s.wait_event(t0)
        ends = []
        for i in range(nch):
            a, b = n * i // nch, n * (i + 1) // nch
            si, so = s_in[i % nstr], s_out[i % nstr]
            with torch.cuda.stream(si):
                xd[a:b].copy_(xh[a:b], non_blocking=True)
                e = ev(); e.record(si)
            so.wait_event(e)
            with torch.cuda.stream(so):
                yh[a:b].copy_(yd[a:b], non_blocking=True)
                e2 = ev(); e2.record(so)
            ends.append(e2)
        torch.cuda.synchronize()
        best = min(best, max(t0.elapsed_time(e) for e in ends))
    return best


for nstr in (1, 2, 4):
    print("streams/direction %d: " % nstr + "  ".join("nch=%d %.3f" % (c, run(c, nstr)) for c in (4, 8, 16, 32)))
