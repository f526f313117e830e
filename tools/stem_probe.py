"""Time the im2col stem conv (fprop + wgrad) at 4x192^3 -> 64 through the C-ABI."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1812_07816_b200 import ops
from paper_1812_07816_b200._native import ALGO_IM2COL, DT_BF16

shape = (1, 192, 192, 192, 4)
rng = np.random.default_rng(0)
x = rng.standard_normal(shape).astype(np.float32)
w = (rng.standard_normal((64, 27, 4)) * 0.1).astype(np.float32)
dy = rng.standard_normal(shape[:4] + (64,)).astype(np.float32)
for kind in ("conv_fwd", "conv_wgrad"):
    for _ in range(2):
        if kind == "conv_fwd":
            ops.conv_op(kind, x=x, w=w, algo=ALGO_IM2COL, dtype=DT_BF16, repeat=5)
        else:
            ops.conv_op(kind, x=x, w=w, dy=dy, algo=ALGO_IM2COL, dtype=DT_BF16, repeat=5)
        print(kind, "%.3f ms" % (1e3 * ops.last_op_seconds()))
