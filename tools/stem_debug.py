import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch, torch.nn.functional as F
from paper_1812_07816_b200 import ops
from paper_1812_07816_b200._native import ALGO_IM2COL, DT_BF16

def bf(a):
    return ops.from_bf16_bits(ops.to_bf16_bits(a)).reshape(a.shape)
shape = (1, 16, 16, 16, 4)
rng = np.random.default_rng(21)
x = bf(rng.standard_normal(shape).astype(np.float32))
w = bf((rng.standard_normal((64, 27, 4)) * 0.1).astype(np.float32))
dy = bf(rng.standard_normal(shape[:4] + (64,)).astype(np.float32))
xt = torch.as_tensor(x, dtype=torch.float64).permute(0, 4, 1, 2, 3).requires_grad_(True)
wt = torch.as_tensor(w, dtype=torch.float64).reshape(64, 3, 3, 3, 4).permute(0, 4, 1, 2, 3).requires_grad_(True)
yt = F.conv3d(xt, wt, padding=1)
yt.backward(torch.as_tensor(dy, dtype=torch.float64).permute(0, 4, 1, 2, 3))
ref_y = yt.permute(0, 2, 3, 4, 1).detach().numpy()
ref_g = wt.grad.permute(0, 2, 3, 4, 1).reshape(64, 27, 4).numpy()
y, part, _ = ops.conv_op("conv_fwd", x=x, w=w, algo=ALGO_IM2COL, dtype=DT_BF16, want_stats=True)
err = np.abs(y - ref_y)
print("fwd max err", err.max(), "ref max", np.abs(ref_y).max())
bad = np.argwhere(err > 0.05 * np.abs(ref_y).max())
print("bad count", len(bad), bad[:10])
nparts = ops.stat_parts_for(shape + (64,))
print("nparts", nparts, "part shape", part.shape)
s = part.reshape(-1)[:nparts * 128].reshape(nparts, 2, 64).sum(0)
print("sum err", np.abs(s[0] - ref_y.reshape(-1, 64).sum(0)).max(), np.abs(ref_y.reshape(-1,64).sum(0)).max())
gw, _ = ops.conv_op("conv_wgrad", x=x, dy=dy, w=w, algo=ALGO_IM2COL, dtype=DT_BF16)
e = np.abs(gw - ref_g)
print("wgrad max err", e.max(), "ref max", np.abs(ref_g).max())
print(np.argwhere(e > 0.01 * np.abs(ref_g).max())[:10])
