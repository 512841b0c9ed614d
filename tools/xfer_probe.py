"""Host-link floor of emrkc_step_host's chunked transfers (no kernels): 4 SoA
rows of nn doubles, K z-chunks, H2D on one stream, D2H of chunk c on another
after H2D of chunk c + 1 (the step's halo dependency)."""
import sys

import torch

nn = 128 ** 3
K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
hin = torch.empty(4, nn, dtype=torch.float64).pin_memory()
hout = torch.empty(4, nn, dtype=torch.float64).pin_memory()
d = torch.empty(4, nn, dtype=torch.float64, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
bounds = [c * nn // K for c in range(K + 1)]


def run(mode):
    ev = [torch.cuda.Event() for _ in range(K)]
    cur = torch.cuda.current_stream()
    s_in.wait_stream(cur)
    s_out.wait_stream(cur)
    for c in range(K):
        a, b = bounds[c], bounds[c + 1]
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s_in):
                for r in range(4):
                    d[r, a:b].copy_(hin[r, a:b], non_blocking=True)
                ev[c].record(s_in)
    for c in range(K):
        a, b = bounds[c], bounds[c + 1]
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s_out):
                if mode == "both":
                    s_out.wait_event(ev[min(c + 1, K - 1)])
                for r in range(4):
                    hout[r, a:b].copy_(d[r, a:b], non_blocking=True)
    cur.wait_stream(s_in)
    cur.wait_stream(s_out)


for mode in ("h2d", "d2h", "both"):
    for _ in range(3):
        run(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        run(mode)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"K={K} {mode}: {ms:.3f} ms per step-equivalent")
