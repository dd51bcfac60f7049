"""PCIe bandwidth of this GPU from pinned host memory: H2D alone, D2H alone, and both at once
on two streams (the e2e bench's steady state).  Prints one JSON line (GB/s)."""
import json

import torch

n = 4 << 30  # bytes per copy
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        a.record()
        fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_gbs": n / t1 / 1e9, "d2h_gbs": n / t2 / 1e9, "duplex_total_gbs": 2 * n / t3 / 1e9,
                  "bytes_per_copy": n}))
