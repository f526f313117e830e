"""One training step of a bench config (for ncu launch lists).

    python tools/step_probe.py f192-c4
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "f192-c4"
dims, batch, preset, _ = bench.CONFIGS[name]
tr = UNetTrainer(TrainConfig(dims=dims, batch=batch, preset=preset, dtype="bf16"))
x, y = tr.synthetic_batch(seed=0)
out = tr.step(x, y)
print(name, out)
