"""Cost of cudaEventRecord between small kernels while a D2H copy saturates PCIe."""
import torch

dev = torch.device("cuda:0")
small = torch.zeros(1 << 20, device=dev)
big = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
host = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True)
s_comp = torch.cuda.Stream()
s_copy = torch.cuda.Stream()


def run(copy, events):
    torch.cuda.synchronize()
    if copy:
        with torch.cuda.stream(s_copy):
            for _ in range(3):
                host.copy_(big, non_blocking=True)
    evs = [torch.cuda.Event(enable_timing=(events == "timing")) for _ in range(400)] if events else []
    with torch.cuda.stream(s_comp):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(400):
            small.add_(1.0)
            if events:
                evs[i].record()
        b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 400 * 1e3


for events in (None, "timing", "notiming"):
    for copy in (False, True):
        run(copy, events)
        print("events=%-8s copy=%-5s %.1f us per kernel" % (events, copy, run(copy, events)))
