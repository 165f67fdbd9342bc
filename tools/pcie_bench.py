"""PCIe copy throughput on the box (tool): pinned H2D, D2H, both directions concurrently."""
import torch
n = 64 * 1024 * 1024  # 256 MB
h = torch.empty(n, pin_memory=True)
h2 = torch.empty(n, pin_memory=True)
d = torch.empty(n, device="cuda")
d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)
def h2d():
    d.copy_(h, non_blocking=True)
def d2h():
    h.copy_(d, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for name, fn, by in [("h2d", h2d, n * 4), ("d2h", d2h, n * 4), ("both", both, 2 * n * 4)]:
    ms = timed(fn)
    print(f"{name}: {ms:.2f} ms, {by / ms / 1e6:.1f} GB/s")
