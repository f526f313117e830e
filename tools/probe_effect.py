"""Does a previously created (and closed) trainer slow a later one?  Times a no-swap
192^3 step with and without a probe trainer run first in the same process."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer


def timed(tr, k=5):
    x, y = tr.synthetic_batch(seed=0)
    tr.load_batch(x, y)
    for _ in range(3):
        tr.step()
    tr.engine.mark(0)
    for _ in range(k):
        tr.run_async()
    tr.engine.mark(1)
    t = tr.engine.elapsed()
    tr.engine.sync()
    return 1e3 * t / k


mode = sys.argv[1]
cfg = dict(dims=(192, 192, 192), preset=None)
if mode == "probe":
    p = UNetTrainer(TrainConfig(**cfg))
    print("probe", timed(p))
    p.close()
    del p
tr = UNetTrainer(TrainConfig(**cfg))
print(mode, "main", timed(tr))
