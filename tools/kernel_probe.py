"""Run one tcgen05 conv kernel at a production shape (for ncu captures).

    python tools/kernel_probe.py conv_fwd 1 192 192 192 64 64 [split]

split (conv_fwd / conv_wgrad): read the input as two sources, channels [0, split) and
[split, Cin) (the dual-source concat of the synthesis conv1).
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1812_07816_b200 import ops  # noqa: E402
from paper_1812_07816_b200._native import ALGO_TCGEN05, DT_BF16  # noqa: E402

kind = sys.argv[1]
n, d, h, w, cin, cout = (int(v) for v in sys.argv[2:8])
rng = np.random.default_rng(0)
w_ = (rng.standard_normal((cout, 27, cin)) * 0.05).astype(np.float32)
if kind.startswith("convt"):
    x = rng.standard_normal((n, d, h, w, cin), dtype=np.float32)
    dy = rng.standard_normal((n, 2 * d, 2 * h, 2 * w, cout), dtype=np.float32)
else:
    x = rng.standard_normal((n, d, h, w, cin), dtype=np.float32)
    dy = rng.standard_normal((n, d, h, w, cout), dtype=np.float32)
args = dict(w=w_, algo=ALGO_TCGEN05, dtype=DT_BF16, repeat=2)
split = int(sys.argv[8]) if len(sys.argv) > 8 else 0
if split:
    x, args["x2"] = np.ascontiguousarray(x[..., :split]), np.ascontiguousarray(x[..., split:])
if kind.endswith("fwd"):
    args["x"] = x
elif kind.endswith("dgrad"):
    args["dy"] = dy
else:
    args["x"], args["dy"] = x, dy
out = ops.conv_op(kind, **args)
t = ops.last_op_seconds()
flops = 2.0 * 27 * n * d * h * w * cin * cout * (8 if kind.startswith("convt") else 1)
print(f"{kind} {n}x{d}x{h}x{w} {cin}->{cout}{' split ' + str(split) if split else ''}: "
      f"{t * 1e3:.3f} ms  {flops / t / 1e12:.1f} TFLOP/s")
