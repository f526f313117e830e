"""Do PCIe copies on a side stream slow small kernels on the compute stream?
Times 400 small elementwise kernels alone, during a D2H copy and during an H2D copy."""
import torch

dev = torch.device("cuda:0")
small = torch.zeros(1 << 20, device=dev)
big = torch.empty(2 << 30, dtype=torch.uint8, device=dev)
host = torch.empty(2 << 30, dtype=torch.uint8, pin_memory=True)
s_comp = torch.cuda.Stream()
s_copy = torch.cuda.Stream()


def run(kind):
    torch.cuda.synchronize()
    if kind == "d2h":
        with torch.cuda.stream(s_copy):
            host.copy_(big, non_blocking=True)
    elif kind == "h2d":
        with torch.cuda.stream(s_copy):
            big.copy_(host, non_blocking=True)
    with torch.cuda.stream(s_comp):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(400):
            small.add_(1.0)
        b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 400 * 1e3


for kind in ("alone", "d2h", "h2d", "alone"):
    run(kind)
    print(kind, "%.1f us per small kernel" % run(kind))
