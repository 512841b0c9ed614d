"""Host link bandwidth: H2D, D2H and both at once (pinned, 64 MiB)."""
import torch

n = 8 << 20
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d1.copy_(h1, non_blocking=True)
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()


def t(f, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


b = 8 * n / 1e9
th = t(lambda: d1.copy_(h1, non_blocking=True))
td = t(lambda: h2.copy_(d2, non_blocking=True))
tb = t(both)
print(f"H2D {b / th * 1e3:.1f} GB/s  D2H {b / td * 1e3:.1f} GB/s  both {2 * b / tb * 1e3:.1f} GB/s "
      f"({th:.3f} / {td:.3f} / {tb:.3f} ms per 64 MiB)")
