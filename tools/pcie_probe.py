"""Host<->device copy bandwidth of the swap engine's binding resource (PCIe), pinned host
memory: each direction alone and both at once, with 1 / 2 / 4 streams per direction and
chunked copies, to see whether more copy engines in flight raise the duplex rate."""
import json
import sys
import time

import torch

n = int(float(sys.argv[1]) * (1 << 30)) if len(sys.argv) > 1 else 1 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def copies(direction, ns, chunks, base):
    step = n // chunks
    for c in range(chunks):
        s = streams[base + c % ns]
        with torch.cuda.stream(s):
            sl = slice(c * step, (c + 1) * step)
            if direction == "d2h":
                h1[sl].copy_(d1[sl], non_blocking=True)
            else:
                d2[sl].copy_(h2[sl], non_blocking=True)


out = {"bytes": n}
for ns, chunks in ((1, 1), (1, 8), (2, 8), (4, 16)):
    key = f"s{ns}_c{chunks}"
    out[f"d2h_{key}"] = n / timed(lambda: copies("d2h", ns, chunks, 0)) / 1e9
    out[f"h2d_{key}"] = n / timed(lambda: copies("h2d", ns, chunks, 4)) / 1e9
    out[f"duplex_{key}"] = n / timed(lambda: (copies("d2h", ns, chunks, 0),
                                             copies("h2d", ns, chunks, 4))) / 1e9
print(json.dumps(out))
