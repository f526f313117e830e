"""Step time of the no-swap 192^3 step alone vs. with a background PCIe copy stream."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer

graph = sys.argv[1] == "graph" if len(sys.argv) > 1 else True
tr = UNetTrainer(TrainConfig(dims=(192, 192, 192), preset=None, graph=graph))
x, y = tr.synthetic_batch(seed=0)
tr.load_batch(x, y)
for _ in range(4):
    tr.step()
big = torch.empty(4 << 30, dtype=torch.uint8, device="cuda:0")
host = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True)
s_copy = torch.cuda.Stream()


def timed(k=5):
    tr.engine.mark(0)
    for _ in range(k):
        tr.run_async()
    tr.engine.mark(1)
    t = tr.engine.elapsed()
    tr.engine.sync()
    return 1e3 * t / k


print("alone", timed())
for kind in ("d2h", "h2d"):
    torch.cuda.synchronize()
    with torch.cuda.stream(s_copy):
        for _ in range(8):
            if kind == "d2h":
                host.copy_(big, non_blocking=True)
            else:
                big.copy_(host, non_blocking=True)
    print(kind, timed())
    torch.cuda.synchronize()
print("alone", timed())


def by_kind(rows):
    acc = {}
    for _, name, _, t in rows:
        acc[name] = acc.get(name, 0.0) + 1e3 * t
    return acc


base = by_kind(tr.op_times(2))
torch.cuda.synchronize()
with torch.cuda.stream(s_copy):
    for _ in range(12):
        host.copy_(big, non_blocking=True)
busy = by_kind(tr.op_times(2))
torch.cuda.synchronize()
for k in sorted(base, key=lambda k: -base[k]):
    print("%-12s %8.3f %8.3f ms" % (k, base[k], busy.get(k, 0.0)))
