import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1812_07816_b200 import ops
from paper_1812_07816_b200._native import ALGO_IM2COL, DT_BF16
shape = (1, 16, 16, 16, 4)
rng = np.random.default_rng(0)
x = rng.standard_normal(shape).astype(np.float32)
w = (rng.standard_normal((64, 27, 4)) * 0.1).astype(np.float32)
dy = rng.standard_normal(shape[:4] + (64,)).astype(np.float32)
which = sys.argv[1] if len(sys.argv) > 1 else "fwd"
if which == "fwd":
    y, _ = ops.conv_op("conv_fwd", x=x, w=w, algo=ALGO_IM2COL, dtype=DT_BF16)
    print("fwd ok", float(np.abs(y).max()))
else:
    g, _ = ops.conv_op("conv_wgrad", x=x, w=w, dy=dy, algo=ALGO_IM2COL, dtype=DT_BF16)
    print("wgrad ok", float(np.abs(g).max()))
