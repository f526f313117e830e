"""The tiny configuration under compute-sanitizer (race detection / sanitizers):
one toy-mode step (reference run_numeric arithmetic, paper-c1, 8^3) and two real-op steps of a
32^3 depth-3 U-Net with every cross-phase tensor swapped (paper-c1) and poison mode on, eager
(no CUDA graph) so the tool sees every launch.

    compute-sanitizer --tool memcheck --error-exitcode 99 python tools/sanitize_tiny.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1812_07816_b200 import numeric  # noqa: E402
from paper_1812_07816_b200.models import UNetParams, gen_unet3d  # noqa: E402
from paper_1812_07816_b200.rewrite import apply_rewrite, resolve_preset  # noqa: E402
from paper_1812_07816_b200.training import expand_training_graph  # noqa: E402
from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer  # noqa: E402

p = UNetParams(dims=(8, 8, 8), in_channels=1, base_filters=1, depth=2, convs_per_level=1)
tg = expand_training_graph(gen_unet3d(p))
rw, plan = apply_rewrite(tg, resolve_preset("paper-c1"))
loss, grads = numeric.run_numeric(rw, plan, seed=1)
print(f"toy loss {loss:.6f}")
cfg = TrainConfig(dims=(32, 32, 32), base_filters=16, depth=3, dtype="bf16",
                  preset="paper-c1", graph=False, poison=True)
tr = UNetTrainer(cfg)
x, y = tr.synthetic_batch(seed=1)
for _ in range(2):
    out = tr.step(x, y)
assert np.isfinite(out["loss"]), out["loss"]
print(f"unet loss {out['loss']:.6f}, swapped {out['d2h_bytes']} B")
