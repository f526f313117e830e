"""GPU: every convolution kernel (tcgen05 and CUDA-core) against a torch CPU
reference of the same op on bf16-representable inputs.

Tolerances: bf16 outputs 1e-2 of max|ref| (output rounding), and every bf16 output
element within one bf16 ulp of the fp64 result (fp32 accumulation in the tensor-core
kernels); fp32 outputs (weight gradients, fp32 check mode) 1e-4 / 1e-5 of max|ref|."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_1812_07816_b200 import ops
from paper_1812_07816_b200._native import ALGO_DIRECT, ALGO_IM2COL, ALGO_TCGEN05, DT_BF16, DT_F32

pytestmark = pytest.mark.gpu


def bf(a):
    return ops.from_bf16_bits(ops.to_bf16_bits(a)).reshape(a.shape)


def rand(shape, seed, scale=1.0):
    return bf(np.random.default_rng(seed).standard_normal(shape).astype(np.float32) * scale)


def t_x(a):    # NDHWC -> NCDHW torch
    return torch.as_tensor(a, dtype=torch.float64).permute(0, 4, 1, 2, 3)


def t_conv_w(w):
    cout, _, cin = w.shape
    return torch.as_tensor(w, dtype=torch.float64).reshape(cout, 3, 3, 3, cin).permute(0, 4, 1, 2, 3)


def t_convt_w(w):
    cout, _, cin = w.shape
    return torch.as_tensor(w, dtype=torch.float64).reshape(cout, 3, 3, 3, cin).permute(4, 0, 1, 2, 3)


def to_ndhwc(t):
    return t.permute(0, 2, 3, 4, 1).detach().numpy()


def ref_conv(x, w, dy=None):
    xt = t_x(x).requires_grad_(True)
    wt = t_conv_w(w).requires_grad_(True)
    y = F.conv3d(xt, wt, padding=1)
    if dy is None:
        return to_ndhwc(y)
    y.backward(t_x(dy))
    g = wt.grad.permute(0, 2, 3, 4, 1).reshape(w.shape).numpy()
    return to_ndhwc(y), to_ndhwc(xt.grad), g


def ref_convt(x, w, dy=None):
    xt = t_x(x).requires_grad_(True)
    wt = t_convt_w(w).requires_grad_(True)
    y = F.conv_transpose3d(xt, wt, stride=2, padding=1, output_padding=1)
    if dy is None:
        return to_ndhwc(y)
    y.backward(t_x(dy))
    g = wt.grad.permute(1, 2, 3, 4, 0).reshape(w.shape).numpy()
    return to_ndhwc(y), to_ndhwc(xt.grad), g


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-12))


CONV_SHAPES = [  # N, D, H, W, Cin, Cout
    (1, 16, 16, 16, 64, 64),
    (1, 12, 12, 12, 128, 256),
    (1, 16, 16, 16, 16, 64),
    (2, 8, 8, 8, 32, 32),
    (1, 8, 8, 8, 256, 128),
    (1, 6, 6, 6, 64, 512),
    # halo-tile path (W >= 32, H >= 16, channels multiple of 64)
    (1, 4, 16, 32, 64, 64),
    (1, 3, 20, 40, 128, 128),
    (2, 2, 16, 32, 64, 256),
    (1, 2, 32, 64, 256, 64),
    # z-pair halo path (64 output channels): odd depth, ragged H/W tiles, batch 2
    (1, 3, 20, 40, 128, 64),
    (2, 5, 16, 32, 64, 64),
    (1, 1, 16, 40, 64, 64),   # odd tile count: the CTA-pair fprop's last peer tile is a dummy
    (1, 1, 16, 40, 128, 128),  # same for the 128-channel CTA-pair halo kernel
    (1, 5, 5, 5, 64, 64),      # one M tile: the CTA-pair per-tap fprop's peer is a dummy
    (1, 6, 6, 6, 256, 256),    # CTA-pair per-tap weight gradient (two 128-row co blocks)
    (1, 4, 4, 4, 512, 512),
    # depth-5 / base-64 layers at 192^3 (L4 / bottleneck at 12^3, synthesis/l3 at 24^3):
    # split-K over taps at K = 27,648, four N tiles of the pair per-tap kernels
    (1, 12, 12, 12, 1024, 1024),
    (1, 12, 12, 12, 512, 1024),
    (1, 24, 24, 24, 1024, 512),
    (1, 24, 24, 24, 512, 512),
]


def bf16_ulp(a):
    """Spacing of bfloat16 numbers at |a| (8 significant bits)."""
    a = np.abs(np.asarray(a, np.float64))
    e = np.floor(np.log2(np.maximum(a, 1e-30)))
    return np.exp2(e - 7)


def assert_within_one_ulp(y, ref, k=13824):
    """bf16 output vs the fp64 result: at most one bf16 ulp away (a correctly rounded
    value is within half an ulp; fp32 accumulation may land on the other neighbour),
    plus 1e-5 of max|ref| absolute for results that cancel to near zero -- scaled with
    the reduction length k beyond 13,824 (the tensor cores' fp32 accumulation truncates,
    so its error grows with the number of K steps)."""
    err = np.abs(np.asarray(y, np.float64) - ref)
    lim = bf16_ulp(ref) + 1e-5 * max(1.0, k / 13824) * np.abs(ref).max()
    bad = err > lim
    assert not bad.any(), (int(bad.sum()), float((err / lim).max()))


@pytest.mark.parametrize("shape", CONV_SHAPES, ids=str)
def test_conv_fwd_tc(shape):
    n, d, h, w_, cin, cout = shape
    x = rand((n, d, h, w_, cin), 1)
    w = rand((cout, 27, cin), 2, (2.0 / (27 * cin)) ** 0.5)
    y, part, _ = ops.conv_op("conv_fwd", x=x, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16,
                             want_stats=True)
    ref = ref_conv(x, w)
    assert rel(y, ref) < 1e-2
    assert_within_one_ulp(y, ref, k=27 * cin)
    s = part.sum(axis=0)
    flat = ref.reshape(-1, cout)
    assert np.allclose(s[0], flat.sum(0), rtol=2e-3, atol=1e-2 * np.abs(flat).max())
    assert np.allclose(s[1], (flat ** 2).sum(0), rtol=2e-3)


@pytest.mark.parametrize("shape", [s for s in CONV_SHAPES if s[4] % 64 == 0], ids=str)
def test_conv_dgrad_tc(shape):
    n, d, h, w_, cin, cout = shape
    x = rand((n, d, h, w_, cin), 3)
    w = rand((cout, 27, cin), 4, (2.0 / (27 * cin)) ** 0.5)
    dy = rand((n, d, h, w_, cout), 5)
    dx, _ = ops.conv_op("conv_dgrad", dy=dy, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    _, ref_dx, _ = ref_conv(x, w, dy)
    assert rel(dx, ref_dx) < 1e-2
    assert_within_one_ulp(dx, ref_dx, k=27 * cout)


@pytest.mark.parametrize("shape", [s for s in CONV_SHAPES if s[4] % 64 == 0 and s[5] % 64 == 0],
                         ids=str)
def test_conv_wgrad_tc(shape):
    n, d, h, w_, cin, cout = shape
    x = rand((n, d, h, w_, cin), 6)
    w = rand((cout, 27, cin), 7, 0.05)
    dy = rand((n, d, h, w_, cout), 8)
    gw, _ = ops.conv_op("conv_wgrad", x=x, dy=dy, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    _, _, ref_g = ref_conv(x, w, dy)
    # fp32 accumulation of bf16-exact products over up to 13,824 voxels
    assert rel(gw, ref_g) < 1e-4


def test_conv_wgrad_tc_narrow_input():
    # 32-channel padded input layer: A operand as 4 taps x 32 channels (SWIZZLE_64B MN-major)
    x = rand((1, 16, 16, 16, 32), 17)
    w = rand((64, 27, 32), 18, 0.05)
    dy = rand((1, 16, 16, 16, 64), 19)
    gw, _ = ops.conv_op("conv_wgrad", x=x, dy=dy, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    _, _, ref_g = ref_conv(x, w, dy)
    assert rel(gw, ref_g) < 1e-4
    y, _ = ops.conv_op("conv_fwd", x=x, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    assert rel(y, ref_conv(x, w)) < 1e-2


@pytest.mark.parametrize("shape", [(1, 16, 16, 16, 4, 64), (2, 8, 8, 32, 4, 64),
                                   (1, 3, 4, 96, 4, 64), (1, 5, 8, 48, 4, 64)], ids=str)
def test_conv_stem_im2col(shape):
    # 4-modality input layer: one tcgen05 GEMM (K = 27*4 padded to 128) over an im2col
    # tile built in shared memory; forward with BN partial sums (Gram-matrix statistics)
    # and the weight gradient.  Both tile boxes (32x4, 16x8) are exercised.
    n, d, h, w_, cin, cout = shape
    x = rand((n, d, h, w_, cin), 21)
    w = rand((cout, 27, cin), 22, (2.0 / (27 * cin)) ** 0.5)
    dy = rand((n, d, h, w_, cout), 23)
    y, part, _ = ops.conv_op("conv_fwd", x=x, w=w, algo=ALGO_IM2COL, dtype=DT_BF16,
                             want_stats=True)
    ref_y, _, ref_g = ref_conv(x, w, dy)
    assert rel(y, ref_y) < 1e-2
    assert_within_one_ulp(y, ref_y)
    nparts = ops.stat_parts_for(shape)
    s = part.reshape(-1)[:nparts * 2 * cout].reshape(nparts, 2, cout).sum(axis=0)
    flat = ref_y.reshape(-1, cout)
    assert np.allclose(s[0], flat.sum(0), rtol=2e-3, atol=1e-2 * np.abs(flat).max())
    assert np.allclose(s[1], (flat ** 2).sum(0), rtol=2e-3)
    gw, _ = ops.conv_op("conv_wgrad", x=x, dy=dy, w=w, algo=ALGO_IM2COL, dtype=DT_BF16)
    assert rel(gw, ref_g) < 1e-4


@pytest.mark.parametrize("kind,shape", [("conv", (1, 4, 16, 32, 64, 64)),
                                        ("conv", (1, 8, 8, 8, 256, 128)),
                                        ("convt", (1, 6, 6, 6, 256, 128))], ids=str)
def test_dgrad_fused_relu_mask(kind, shape):
    # ReLU backward fused into the dgrad epilogue: dx = dgrad * (act > 0)
    n, d, h, w_, cin, cout = shape
    up = 2 if kind == "convt" else 1
    x = rand((n, d, h, w_, cin), 31)
    w = rand((cout, 27, cin), 32, (2.0 / (27 * cin)) ** 0.5)
    dy = rand((n, d * up, h * up, w_ * up, cout), 33)
    act = np.maximum(rand((n, d, h, w_, cin), 34), 0.0)
    dx, _ = ops.conv_op(kind + "_dgrad", dy=dy, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16,
                        relu_mask=act)
    ref_fn = ref_convt if kind == "convt" else ref_conv
    _, ref_dx, _ = ref_fn(x, w, dy)
    ref_dx = ref_dx * (act > 0)
    assert rel(dx, ref_dx) < 1e-2
    assert np.all(dx[act <= 0] == 0)


CONVT_SHAPES = [  # N, Dl, Hl, Wl, Cin, Cout
    (1, 8, 8, 8, 128, 64),
    (1, 6, 6, 6, 256, 128),
    (2, 4, 4, 4, 512, 256),
    (1, 3, 5, 7, 128, 64),
    (1, 12, 12, 12, 1024, 512),   # depth-5 synthesis/l3 upsample at 192^3
]


@pytest.mark.parametrize("shape", CONVT_SHAPES, ids=str)
def test_convt_tc(shape):
    n, d, h, w_, cin, cout = shape
    x = rand((n, d, h, w_, cin), 9)
    w = rand((cout, 27, cin), 10, (2.0 / (27 * cin)) ** 0.5)
    dy = rand((n, 2 * d, 2 * h, 2 * w_, cout), 11)
    ref_y, ref_dx, ref_g = ref_convt(x, w, dy)
    y, _ = ops.conv_op("convt_fwd", x=x, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    assert rel(y, ref_y) < 1e-2
    assert_within_one_ulp(y, ref_y)
    dx, _ = ops.conv_op("convt_dgrad", dy=dy, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    assert rel(dx, ref_dx) < 1e-2
    assert_within_one_ulp(dx, ref_dx)
    gw, _ = ops.conv_op("convt_wgrad", x=x, dy=dy, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    assert rel(gw, ref_g) < 1e-4


@pytest.mark.parametrize("shape", [
    (1, 3, 5, 7, 64, 32),     # sub-pixel GEMM, ragged low-res grid, N' = 8 Cout = 256
    (1, 4, 4, 4, 32, 16),     # 8-launch parity-class fallback (Cin % 64 != 0)
], ids=str)
def test_convt_fwd_paths(shape):
    n, d, h, w_, cin, cout = shape
    x = rand((n, d, h, w_, cin), 17)
    w = rand((cout, 27, cin), 18, (2.0 / (27 * cin)) ** 0.5)
    dy = rand((n, 2 * d, 2 * h, 2 * w_, cout), 19)
    ref_y, _, _ = ref_convt(x, w, dy)
    y, _ = ops.conv_op("convt_fwd", x=x, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    assert rel(y, ref_y) < 1e-2


@pytest.mark.parametrize("shape", [(1, 6, 6, 6, 4, 8), (2, 4, 4, 4, 8, 16)], ids=str)
def test_direct_kernels_fp32(shape):
    n, d, h, w_, cin, cout = shape
    x = rand((n, d, h, w_, cin), 12)
    w = rand((cout, 27, cin), 13, 0.2)
    dy = rand((n, d, h, w_, cout), 14)
    ref_y, ref_dx, ref_g = ref_conv(x, w, dy)
    y, _ = ops.conv_op("conv_fwd", x=x, w=w, algo=ALGO_DIRECT, dtype=DT_F32)
    dx, _ = ops.conv_op("conv_dgrad", dy=dy, w=w, algo=ALGO_DIRECT, dtype=DT_F32)
    gw, _ = ops.conv_op("conv_wgrad", x=x, dy=dy, w=w, algo=ALGO_DIRECT, dtype=DT_F32)
    assert rel(y, ref_y) < 1e-5 and rel(dx, ref_dx) < 1e-5 and rel(gw, ref_g) < 1e-5
    wt = rand((cout, 27, cin), 15, 0.2)
    dyt = rand((n, 2 * d, 2 * h, 2 * w_, cout), 16)
    ref_y, ref_dx, ref_g = ref_convt(x, wt, dyt)
    y, _ = ops.conv_op("convt_fwd", x=x, w=wt, algo=ALGO_DIRECT, dtype=DT_F32)
    dx, _ = ops.conv_op("convt_dgrad", dy=dyt, w=wt, algo=ALGO_DIRECT, dtype=DT_F32)
    gw, _ = ops.conv_op("convt_wgrad", x=x, dy=dyt, w=wt, algo=ALGO_DIRECT, dtype=DT_F32)
    assert rel(y, ref_y) < 1e-5 and rel(dx, ref_dx) < 1e-5 and rel(gw, ref_g) < 1e-5


def ref_loss(act, labels, hw, hb, relu, eps=1e-5):
    """float64 head + softmax + soft Dice forward/backward (unet.py DICE loss)."""
    c = act.shape[-1]
    a = act.reshape(-1, c).astype(np.float64)
    g = labels.ravel().astype(np.int64)
    ncls = hw.shape[0]
    z = a @ hw.T.astype(np.float64) + hb
    z -= z.max(1, keepdims=True)
    p = np.exp(z)
    p /= p.sum(1, keepdims=True)
    oh = np.eye(ncls)[g]
    I, P, G = (p * oh).sum(0), p.sum(0), oh.sum(0)
    den = P + G + eps
    loss = 1.0 - np.mean((2 * I + eps) / den)
    dp = oh * (-(2.0 / ncls) / den) + (1.0 / ncls) * (2 * I + eps) / den ** 2
    dz = p * (dp - (p * dp).sum(1, keepdims=True))
    dact = dz @ hw.astype(np.float64)
    if relu:
        dact = dact * (a > 0)
    return I, P, G, loss, dact.reshape(act.shape), dz.T @ a, dz.sum(0)


@pytest.mark.parametrize("case", [
    ((1, 5, 7, 9), 64, 4, True),     # tiled fwd / octet bwd bf16 kernels, ragged tail
    ((2, 8, 8, 8), 64, 3, False),
    ((1, 4, 6, 6), 16, 4, True),     # thread-per-voxel kernel (C < 64)
], ids=str)
def test_loss_kernels(case):
    grid, c, ncls, relu = case
    rng = np.random.default_rng(21)
    act = ops.from_bf16_bits(ops.to_bf16_bits(
        rng.standard_normal(grid + (c,)).astype(np.float32)))
    labels = rng.integers(0, ncls, size=grid)
    hw = (rng.standard_normal((ncls, c)) * 0.2).astype(np.float32)
    hb = (rng.standard_normal(ncls) * 0.1).astype(np.float32)
    dice, dact, ghw, ghb = ops.loss_op(act, labels, hw, hb, relu=relu)
    I, P, G, loss, rdact, rghw, rghb = ref_loss(act, labels, hw, hb, relu)
    assert np.allclose(dice[:ncls], I, rtol=1e-4)
    assert np.allclose(dice[ncls:2 * ncls], P, rtol=1e-4)
    assert np.array_equal(dice[2 * ncls:3 * ncls], G)
    assert abs(dice[3 * ncls] - loss) < 1e-5
    assert rel(dact, rdact) < 1e-2
    if relu:
        assert np.all(dact[act <= 0] == 0)
    assert rel(ghw, rghw) < 1e-3
    assert rel(ghb, rghb) < 1e-3


def test_halo_64_column_fallback_kernel():
    """The 8x16x1 halo kernel for 64 output channels (replaced by the z-pair kernel,
    kept behind US_NO_Z2=1) still matches the reference."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, sys\n"
        "sys.path.insert(0, 'tests')\n"
        "from test_gpu_kernels import rand, ref_conv, rel, ops, ALGO_TCGEN05, DT_BF16\n"
        "x = rand((1, 3, 16, 32, 128), 1); w = rand((64, 27, 128), 2, (2.0 / 3456) ** 0.5)\n"
        "dy = rand((1, 3, 16, 32, 64), 3)\n"
        "y, _ = ops.conv_op('conv_fwd', x=x, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)\n"
        "assert rel(y, ref_conv(x, w)) < 1e-2\n"
        "w2 = rand((128, 27, 64), 4, (2.0 / 1728) ** 0.5); x2 = rand((1, 3, 16, 32, 64), 5)\n"
        "dy2 = rand((1, 3, 16, 32, 128), 6)\n"
        "dx, _ = ops.conv_op('conv_dgrad', dy=dy2, w=w2, algo=ALGO_TCGEN05, dtype=DT_BF16)\n"
        "assert rel(dx, ref_conv(x2, w2, dy2)[1]) < 1e-2\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env=dict(os.environ, US_NO_Z2="1"), timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_loss_kernel_variants_agree(tmp_path):
    """The octet backward (default) and the smem-tiled backward (US_LOSS_TILE=1, also the
    fused-BN-sums path) compute the same head gradients and dact."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, sys\n"
        "sys.path.insert(0, 'tests')\n"
        "from test_gpu_kernels import ops\n"
        "rng = np.random.default_rng(5)\n"
        "act = ops.from_bf16_bits(ops.to_bf16_bits(rng.standard_normal((2, 9, 10, 11, 64)).astype(np.float32)))\n"
        "lab = rng.integers(0, 4, size=(2, 9, 10, 11))\n"
        "hw = (rng.standard_normal((4, 64)) * 0.2).astype(np.float32); hb = np.zeros(4, np.float32)\n"
        "d, dact, ghw, ghb = ops.loss_op(act, lab, hw, hb, relu=True)\n"
        "np.save(sys.argv[1], np.concatenate([dact.ravel(), ghw.ravel(), ghb.ravel()]))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    tmp = str(tmp_path)
    for i, env in enumerate(({}, {"US_LOSS_TILE": "1"})):
        path = os.path.join(tmp, f"loss_variant_{i}.npy")
        r = subprocess.run([sys.executable, "-c", code, path], cwd=root, capture_output=True,
                           text=True, env=dict(os.environ, **env), timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert rel(outs[0], outs[1]) < 1e-4


def test_cta_pair_kernels_match_single_cta_bitwise(tmp_path):
    """The CTA-pair (cta_group::2) kernels accumulate every output in the same K order as
    their single-CTA counterparts (US_NO_Z2_PAIR=1), so all outputs agree bit for bit."""
    import os
    import subprocess
    import sys
    cases = [  # kind, N, D, H, W, Cin, Cout
        ("conv_fwd", 1, 3, 16, 32, 64, 64), ("conv_dgrad", 1, 3, 16, 32, 64, 64),
        ("conv_fwd", 1, 2, 16, 32, 128, 128), ("conv_dgrad", 1, 2, 16, 32, 128, 128),
        ("conv_fwd", 1, 2, 16, 32, 128, 256), ("conv_dgrad", 1, 2, 16, 32, 256, 128),
        ("conv_wgrad", 1, 2, 16, 32, 128, 64), ("conv_wgrad", 1, 6, 6, 6, 256, 256),
        ("conv_fwd", 1, 6, 6, 6, 256, 256), ("conv_dgrad", 1, 6, 6, 6, 256, 256),
        # depth-5 layers: four N tiles of the pair per-tap kernels, split-K at K = 27,648
        ("conv_fwd", 1, 12, 12, 12, 1024, 1024), ("conv_dgrad", 1, 12, 12, 12, 1024, 1024),
        ("conv_wgrad", 1, 12, 12, 12, 1024, 1024), ("conv_fwd", 1, 12, 12, 12, 512, 1024),
        ("conv_dgrad", 1, 24, 24, 24, 512, 512), ("conv_fwd", 1, 24, 24, 24, 1024, 512),
    ]
    code = (
        "import numpy as np, sys\n"
        "sys.path.insert(0, 'tests')\n"
        "from test_gpu_kernels import rand, ops, ALGO_TCGEN05, DT_BF16\n"
        "outs = []\n"
        f"for kind, n, d, h, w_, cin, cout in {cases!r}:\n"
        "    x = rand((n, d, h, w_, cin), 1); w = rand((cout, 27, cin), 2, 0.05)\n"
        "    dy = rand((n, d, h, w_, cout), 3)\n"
        "    args = dict(w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)\n"
        "    if kind == 'conv_fwd': args['x'] = x\n"
        "    elif kind == 'conv_dgrad': args['dy'] = dy\n"
        "    else: args['x'], args['dy'] = x, dy\n"
        "    outs.append(ops.conv_op(kind, **args)[0].ravel())\n"
        "np.save(sys.argv[1], np.concatenate(outs))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    tmp = str(tmp_path)
    for i, env in enumerate(({}, {"US_NO_Z2_PAIR": "1"})):
        path = os.path.join(tmp, f"pair_cmp_{i}.npy")
        r = subprocess.run([sys.executable, "-c", code, path], cwd=root, capture_output=True,
                           text=True, env=dict(os.environ, **env), timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(np.load(path))
    assert res[0].shape == res[1].shape
    assert np.array_equal(res[0], res[1])


WGRAD_VARIANT_SHAPES = [  # N, D, H, W, Cin, Cout (+ dual-source split)
    (1, 4, 16, 32, 64, 64, 0), (2, 3, 20, 40, 128, 64, 64), (1, 2, 16, 32, 256, 64, 0),
    (1, 3, 20, 40, 128, 128, 0), (2, 2, 16, 32, 64, 256, 0), (1, 2, 16, 32, 256, 128, 128),
]


@pytest.mark.parametrize("env", [{"US_HV_XA": "1"}, {"US_NO_HV": "1"}], ids=str)
def test_wgrad_kernel_variants_match_fp64(env, tmp_path):
    """Every weight-gradient kernel family (halo-view XA / XB, tap-pair halo, 8-tap halo)
    against the fp64 reference: fp32 accumulation of bf16-exact products, 1e-4 of max."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, sys\n"
        "sys.path.insert(0, 'tests')\n"
        "from test_gpu_kernels import rand, ops, ALGO_TCGEN05, DT_BF16\n"
        "outs = []\n"
        f"for n, d, h, w_, cin, cout, split in {WGRAD_VARIANT_SHAPES!r}:\n"
        "    x = rand((n, d, h, w_, cin), 6); w = rand((cout, 27, cin), 7, 0.05)\n"
        "    dy = rand((n, d, h, w_, cout), 8)\n"
        "    args = dict(w=w, algo=ALGO_TCGEN05, dtype=DT_BF16, dy=dy)\n"
        "    if split: args['x'], args['x2'] = x[..., :split].copy(), x[..., split:].copy()\n"
        "    else: args['x'] = x\n"
        "    outs.append(ops.conv_op('conv_wgrad', **args)[0].ravel())\n"
        "np.save(sys.argv[1], np.concatenate(outs))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(str(tmp_path), "wg.npy")
    r = subprocess.run([sys.executable, "-c", code, path], cwd=root, capture_output=True,
                       text=True, env=dict(os.environ, **env), timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(path)
    off = 0
    for n, d, h, w_, cin, cout, _ in WGRAD_VARIANT_SHAPES:
        x = rand((n, d, h, w_, cin), 6)
        w = rand((cout, 27, cin), 7, 0.05)
        dy = rand((n, d, h, w_, cout), 8)
        _, _, ref_g = ref_conv(x, w, dy)
        g = got[off:off + ref_g.size].reshape(ref_g.shape)
        off += ref_g.size
        assert rel(g, ref_g) < 1e-4, (n, d, h, w_, cin, cout)


DUAL_SHAPES = [  # N, D, H, W, Ca, Cb, Cout: the synthesis conv1 of each U-Net level
    (1, 3, 16, 32, 64, 64, 64),       # L0: z-pair halo fprop, CTA-pair halo wgrad
    (1, 2, 16, 32, 128, 128, 128),    # L1: halo fprop (pair), 8-tap halo wgrad
    (1, 6, 6, 6, 256, 256, 256),      # L2: per-tap fprop (pair), per-tap wgrad (pair)
    (1, 4, 4, 4, 512, 512, 512),      # L3: split-K per-tap fprop
]


@pytest.mark.parametrize("shape", DUAL_SHAPES, ids=str)
def test_dual_source_conv_equals_materialised_concat(shape):
    """The synthesis conv1 reading [skip | upsample] as two TMA sources (the concat never
    written) computes exactly what it computes on the materialised concat: bit-identical
    fprop and weight gradient (same K order)."""
    n, d, h, w_, ca, cb, cout = shape
    xa = rand((n, d, h, w_, ca), 41)
    xb = rand((n, d, h, w_, cb), 42)
    w = rand((cout, 27, ca + cb), 43, (2.0 / (27 * (ca + cb))) ** 0.5)
    dy = rand((n, d, h, w_, cout), 44)
    cat = np.concatenate([xa, xb], axis=-1)
    y1, _ = ops.conv_op("conv_fwd", x=cat, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    y2, _ = ops.conv_op("conv_fwd", x=xa, x2=xb, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    assert np.array_equal(y1, y2)
    assert rel(y2, ref_conv(cat, w)) < 1e-2
    g1, _ = ops.conv_op("conv_wgrad", x=cat, dy=dy, w=w, algo=ALGO_TCGEN05, dtype=DT_BF16)
    g2, _ = ops.conv_op("conv_wgrad", x=xa, x2=xb, dy=dy, w=w, algo=ALGO_TCGEN05,
                        dtype=DT_BF16)
    assert np.array_equal(g1, g2)
