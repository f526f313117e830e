"""Measure host<->device copy bandwidth (pinned, 1 GiB) per direction and both at once."""
import json
import torch

n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        torch.cuda.synchronize()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def d2h():
    with torch.cuda.stream(s1):
        h1.copy_(d1, non_blocking=True)
    s1.synchronize()


def h2d():
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
    s2.synchronize()


def both():
    with torch.cuda.stream(s1):
        h1.copy_(d1, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


out = {"d2h_gbs": n / timed(d2h) / 1e9, "h2d_gbs": n / timed(h2d) / 1e9,
       "bidir_total_gbs": 2 * n / timed(both) / 1e9}
print(json.dumps(out))
