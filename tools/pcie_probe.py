"""Dev probe: pinned H2D / D2H bandwidth alone and concurrently (51 MB, c2's x / y)."""
import torch
n = 51380224 // 4
h1 = torch.empty(n).pin_memory(); h2 = torch.empty(n).pin_memory()
d1 = torch.empty(n, device="cuda"); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
h2d = t(lambda: d1.copy_(h1, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    e = torch.cuda.Event(); e.record()
    s1.wait_event(e); s2.wait_event(e)
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1); e2.record(s2)
    torch.cuda.current_stream().wait_event(e1); torch.cuda.current_stream().wait_event(e2)
bo = t(both)
print("H2D %.3f ms (%.1f GB/s)  D2H %.3f ms (%.1f GB/s)  both %.3f ms" % (h2d, n*4/h2d/1e6, d2h, n*4/d2h/1e6, bo))
