"""torch-CPU fp64 restatement of one real-op U-Net training step -- TEST INFRASTRUCTURE ONLY.

Walks the same graph the engine executes (gen_unet3d, reference
pkg/src/swapsim/models.py:104-159, byte-identical per tests/test_planner_parity.py)
and gives each node kind its real semantics:
  conv      Conv3d k3 s1 p1, no bias (BatchNorm follows)
  norm      BatchNorm3d, batch statistics, biased variance, eps 1e-5
  activation ReLU ; pool MaxPool3d(2) ; upsample ConvTranspose3d k3 s2 p1 op1
  concat    cat([shortcut, upsampled], channels)
  loss      1x1x1 head (+bias) -> softmax -> soft Dice over the batch,
            L = 1 - mean_k (2 I_k + eps) / (P_k + G_k + eps)
followed by one Adam step (Adam, lr 5e-4).  Gradients come from
torch autograd in float64.  Parity of the real-op step is unpinned by the
reference (it has no real-op arithmetic); this oracle is self-consistent and
gradchecked in tests/test_oracle_pinned.py.

Parameter layout shared with the engine: conv/convT weights [Cout][27][Cin]
(tap = kd*9 + kh*3 + kw; the first conv may carry zero-padded input channels),
BN gamma/beta [C], head.w [ncls][C0], head.b [ncls].
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

BN_EPS = 1e-5
DICE_EPS = 1e-5


def conv_w_to_torch(w: np.ndarray, cin_real: int) -> torch.Tensor:
    cout, _, cin = w.shape
    t = torch.as_tensor(np.asarray(w, np.float64)).reshape(cout, 3, 3, 3, cin)[..., :cin_real]
    return t.permute(0, 4, 1, 2, 3).contiguous()


def conv_grad_from_torch(g: torch.Tensor, cin_pad: int) -> np.ndarray:
    cout, cin = g.shape[0], g.shape[1]
    out = np.zeros((cout, 27, cin_pad))
    out[:, :, :cin] = g.permute(0, 2, 3, 4, 1).reshape(cout, 27, cin).detach().numpy()
    return out


def convt_w_to_torch(w: np.ndarray) -> torch.Tensor:
    cout, _, cin = w.shape
    return torch.as_tensor(np.asarray(w, np.float64)).reshape(cout, 3, 3, 3, cin) \
        .permute(4, 0, 1, 2, 3).contiguous()


def convt_grad_from_torch(g: torch.Tensor) -> np.ndarray:
    cin, cout = g.shape[0], g.shape[1]
    return g.permute(1, 2, 3, 4, 0).reshape(cout, 27, cin).detach().numpy()


class _RoundBF16(torch.autograd.Function):
    """Round a value and its incoming gradient to bfloat16 (storage emulation)."""

    @staticmethod
    def forward(ctx, t):
        return t.to(torch.bfloat16).to(t.dtype)

    @staticmethod
    def backward(ctx, g):
        return g.to(torch.bfloat16).to(g.dtype)


def forward_loss(graph, params: dict, x: np.ndarray, y: np.ndarray, n_classes: int,
                 keep=(), dtype=torch.float64, emulate_bf16: bool = False):
    """Returns (loss, leaf tensors by param name, dice sums, kept activations NDHWC).

    emulate_bf16 rounds every stored activation and activation gradient to
    bfloat16 (what the engine's bf16 mode stores), in fp64 arithmetic otherwise:
    the noise floor any bf16-storage implementation is held to."""
    leaves, vals, kept = {}, {}, {}
    npdt = np.float64 if dtype == torch.float64 else np.float32
    rnd = _RoundBF16.apply if emulate_bf16 else (lambda t: t)

    def leaf(name, t):
        t = t.clone().requires_grad_(True)
        leaves[name] = t
        return t

    loss = dice = None
    for n in graph.nodes:
        if n.kind == "source":
            vals[n.outputs[0]] = rnd(torch.as_tensor(np.asarray(x, npdt)))
            continue
        xs = [vals[t] for t in n.inputs]
        if n.kind == "conv":
            cin_real = graph.tensor(n.inputs[0]).channels
            w = leaf(n.id + ".w", conv_w_to_torch(params[n.id + ".w"], cin_real).to(dtype))
            out = F.conv3d(xs[0], w, padding=1)
        elif n.kind == "norm":
            gm = leaf(n.id + ".gamma", torch.as_tensor(np.asarray(params[n.id + ".gamma"],
                                                                  npdt)))
            bt = leaf(n.id + ".beta", torch.as_tensor(np.asarray(params[n.id + ".beta"], npdt)))
            out = F.batch_norm(xs[0], None, None, gm, bt, training=True, eps=BN_EPS)
        elif n.kind == "activation":
            out = F.relu(xs[0])
        elif n.kind == "pool":
            out = F.max_pool3d(xs[0], 2)
        elif n.kind == "upsample":
            w = leaf(n.id + ".w", convt_w_to_torch(params[n.id + ".w"]).to(dtype))
            out = F.conv_transpose3d(xs[0], w, stride=2, padding=1, output_padding=1)
        elif n.kind == "concat":
            out = torch.cat(xs, dim=1)
        elif n.kind == "loss":
            c0 = xs[0].shape[1]
            hw = leaf("head.w", torch.as_tensor(np.asarray(params["head.w"], npdt)))
            hb = leaf("head.b", torch.as_tensor(np.asarray(params["head.b"], npdt)))
            logits = F.conv3d(xs[0], hw.reshape(n_classes, c0, 1, 1, 1), hb)
            p = torch.softmax(logits, dim=1)
            g = F.one_hot(torch.as_tensor(y.astype(np.int64)), n_classes).permute(0, 4, 1, 2, 3)
            g = g.to(dtype)
            inter = (p * g).sum(dim=(0, 2, 3, 4))
            psum = p.sum(dim=(0, 2, 3, 4))
            gsum = g.sum(dim=(0, 2, 3, 4))
            dice_k = (2 * inter + DICE_EPS) / (psum + gsum + DICE_EPS)
            loss = 1 - dice_k.mean()
            dice = torch.cat([inter, psum, gsum]).detach().numpy()
            continue
        else:
            raise ValueError(n.kind)
        if n.kind != "concat":
            out = rnd(out)
        vals[n.outputs[0]] = out
        if n.outputs[0] in keep:
            kept[n.outputs[0]] = out.detach().permute(0, 2, 3, 4, 1).numpy()
    return loss, leaves, dice, kept


def reference_step(cfg, params: dict, x: np.ndarray, y: np.ndarray, keep=(),
                   emulate_bf16: bool = False, dtype=torch.float64) -> dict:
    """One step at fp64: loss, Dice sums, per-parameter grads (engine layout), Adam update.

    dtype=torch.float32 runs the same step in fp32 arithmetic: its distance to the fp64
    step is the conditioning floor any fp32 implementation is held to."""
    from paper_1812_07816_b200.models import gen_unet3d
    torch.set_grad_enabled(True)
    graph = gen_unet3d(cfg.unet_params())
    loss, leaves, dice, kept = forward_loss(graph, params, x, y, cfg.n_classes, keep,
                                            emulate_bf16=emulate_bf16, dtype=dtype)
    loss.backward()
    grads = {}
    for name, t in leaves.items():
        g = t.grad.to(torch.float64)
        if name.endswith(".w") and name != "head.w":
            node = graph.node(name[:-2])
            if node.kind == "conv":
                grads[name] = conv_grad_from_torch(g, params[name].shape[2])
            else:
                grads[name] = convt_grad_from_torch(g)
        else:
            grads[name] = g.detach().numpy().reshape(np.shape(params[name]))
    b1, b2 = cfg.betas
    new = {}
    for name, gr in grads.items():
        m = (1 - b1) * gr
        v = (1 - b2) * gr * gr
        mh, vh = m / (1 - b1), v / (1 - b2)
        new[name] = np.asarray(params[name], np.float64) - cfg.lr * mh / (np.sqrt(vh) + cfg.adam_eps)
    return {"loss": float(loss.detach()), "dice": np.asarray(dice, np.float64), "grads": grads,
            "params_after": new, "acts": {k: np.asarray(v, np.float64) for k, v in kept.items()}}


def init_params(graph, seed: int, n_classes: int) -> dict:
    """The engine's initial parameters (paper_1812_07816_b200/unet.py initial_params,
    fp32 storage -- no padded input channels) rebuilt from the graph alone, so the CPU
    baseline never loads the CUDA library: Kaiming-normal conv / convT weights
    [Cout][27][Cin] from default_rng((seed, crc32(name))), BN gamma 1 / beta 0, head."""
    import zlib
    out = {}
    c0 = None
    for n in graph.nodes:
        if n.kind in ("conv", "upsample"):
            cin = graph.tensor(n.inputs[0]).channels
            cout = graph.tensor(n.outputs[0]).channels
            name = n.id + ".w"
            rng = np.random.default_rng((seed, zlib.crc32(name.encode())))
            out[name] = (rng.standard_normal((cout, 27, cin)) *
                         np.sqrt(2.0 / (27 * cin))).astype(np.float32)
        elif n.kind == "norm":
            c = graph.tensor(n.outputs[0]).channels
            out[n.id + ".gamma"] = np.ones(c, np.float32)
            out[n.id + ".beta"] = np.zeros(c, np.float32)
        elif n.kind == "loss":
            c0 = graph.tensor(n.inputs[0]).channels
    rng = np.random.default_rng((seed, zlib.crc32(b"head.w")))
    out["head.w"] = (rng.standard_normal((n_classes, c0)) * np.sqrt(2.0 / c0)).astype(np.float32)
    out["head.b"] = np.zeros(n_classes, np.float32)
    return out


def synthetic_batch(dims, batch: int, in_channels: int, n_classes: int, seed: int = 0):
    """BraTS-shaped synthetic batch (the engine's recipe, unet.py synthetic_batch; input
    recipe of the reference numeric.py:49-59): N(0,1) fp32 NCDHW volume, uint8 labels."""
    import zlib
    d, h, w = dims
    rng = np.random.default_rng((seed, zlib.crc32(b"source")))
    x = rng.standard_normal(batch * in_channels * d * h * w).astype(np.float32)
    x = x.reshape(batch, in_channels, d, h, w)
    lrng = np.random.default_rng((seed, zlib.crc32(b"label")))
    y = lrng.integers(0, n_classes, size=(batch, d, h, w)).astype(np.uint8)
    return x, y


def cpu_train_step_seconds(cfg, params: dict, x: np.ndarray, y: np.ndarray, steps: int = 2,
                           threads: int | None = None, warmup: int = 0) -> tuple[float, int]:
    """Time the CPU restatement (torch fp32, all host threads): forward, Dice loss,
    backward and an in-place Adam update, after `warmup` untimed steps.  Returns (seconds
    per step -- the best timed step, threads)."""
    import time
    from paper_1812_07816_b200.models import gen_unet3d
    if threads:
        torch.set_num_threads(threads)
    graph = gen_unet3d(cfg.unet_params())
    torch.set_grad_enabled(True)
    state = {}
    times = []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        loss, leaves, _, _ = forward_loss(graph, params, x, y, cfg.n_classes, dtype=torch.float32)
        loss.backward()
        with torch.no_grad():
            for name, t in leaves.items():
                m, v = state.get(name, (torch.zeros_like(t), torch.zeros_like(t)))
                m.mul_(0.9).add_(t.grad, alpha=0.1)
                v.mul_(0.999).addcmul_(t.grad, t.grad, value=0.001)
                state[name] = (m, v)
                t.sub_(cfg.lr * m / (v.sqrt() + cfg.adam_eps))
        if it >= warmup:
            times.append(time.perf_counter() - t0)
    return min(times), torch.get_num_threads()
