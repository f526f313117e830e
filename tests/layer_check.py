"""Per-layer parity of a bf16 training step, teacher-forced on the GPU's own tensors.

A full-step comparison against the fp64 oracle is dominated, at small volumes and
depth 5, by how BatchNorm over a handful of voxels amplifies bf16 storage rounding
(see test_gpu_depth5.py).  This check removes that amplification: every layer's
output is recomputed in fp64 from the inputs the GPU actually stored (captured
activations and activation gradients, the bf16 weights, the saved BatchNorm
statistics) and compared with what the GPU wrote:

  conv / convT forward, conv dgrad (+ fused ReLU mask), convT dgrad   within one bf16 ulp
  BatchNorm + ReLU forward (saved statistics)                           within one bf16 ulp
  BatchNorm backward, loss backward                                     3e-3 relative L2
      (bf16 output rounding alone is ~1.1e-3 RMS; dy - mean(dy) - xhat mean(dy xhat)
      cancels in fp32 before it is rounded)
  max-pool forward / backward, concat                                   exact (tied windows excepted)
  weight gradients (conv, convT), BN gamma/beta, head                   1e-4 relative L2
  batch statistics vs the stored conv output                            1e-2 (from the fp32 output)
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from paper_1812_07816_b200.ops import from_bf16_bits, to_bf16_bits

BN_EPS = 1e-5


def capture_list(graph) -> tuple:
    """Forward tensors and activation gradients the check reads (the upsample output
    and the BN outputs are not requested: capturing them would change the program --
    the upsample writes into its concat, the BN output is dead)."""
    out = []
    for n in graph.nodes:
        if n.kind in ("source", "conv", "activation", "pool", "concat"):
            out.append(n.outputs[0])
        if n.kind in ("conv", "pool", "concat"):
            out.append("d:" + n.outputs[0])
        if n.kind == "norm":
            out.append("d:" + n.outputs[0])
    return tuple(out)


def _t(a):      # NDHWC -> NCDHW float64
    return torch.as_tensor(np.asarray(a, np.float64)).permute(0, 4, 1, 2, 3)


def _nd(t):     # NCDHW -> NDHWC numpy
    return t.detach().permute(0, 2, 3, 4, 1).numpy()


def _bf(a):
    return from_bf16_bits(to_bf16_bits(np.asarray(a, np.float32))).reshape(np.shape(a))


def _ulp(a):
    a = np.abs(np.asarray(a, np.float64))
    return np.exp2(np.floor(np.log2(np.maximum(a, 1e-30))) - 7)


def _rel_l2(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


class LayerCheck:
    def __init__(self, tr, x, y, params):
        self.tr, self.g = tr, tr.graph
        self.x, self.y = x, y
        self.p = params
        self.cap = {}
        self.fail = []
        self.n_checked = 0
        self.stats = tr.bn_stats()
        self.grads = tr.grads_now()

    def c(self, t):
        if t not in self.cap:
            self.cap[t] = self.tr.captured_tensor(t).astype(np.float64)
        return self.cap[t]

    def w_conv(self, nid):   # [Cout][27][Cin] -> torch Conv3d weight, as the kernels read it
        w = _bf(self.p[nid + ".w"]).astype(np.float64)
        cout, _, cin = w.shape
        return torch.as_tensor(w).reshape(cout, 3, 3, 3, cin).permute(0, 4, 1, 2, 3)

    def w_convt(self, nid):  # -> torch ConvTranspose3d weight [Cin][Cout][3][3][3]
        w = _bf(self.p[nid + ".w"]).astype(np.float64)
        cout, _, cin = w.shape
        return torch.as_tensor(w).reshape(cout, 3, 3, 3, cin).permute(4, 0, 1, 2, 3)

    # ------------------------------------------------------------------ assertions
    def ulp(self, what, got, ref, slack=1e-5):
        self.n_checked += 1
        err = np.abs(np.asarray(got, np.float64) - ref)
        lim = _ulp(ref) + slack * max(float(np.abs(ref).max()), 1e-30)
        bad = int((err > lim).sum())
        if bad:
            self.fail.append((what, "ulp", bad, float((err / lim).max())))

    def l2(self, what, got, ref, tol):
        self.n_checked += 1
        e = _rel_l2(got, ref)
        if e > tol:
            self.fail.append((what, "rel_l2", e, tol))

    def exact(self, what, got, ref, skip=None):
        self.n_checked += 1
        d = np.asarray(got, np.float64) != np.asarray(ref, np.float64)
        if skip is not None:
            d &= ~skip
        if d.any():
            self.fail.append((what, "exact", int(d.sum())))

    # ------------------------------------------------------------------ forward
    def forward(self):
        g = self.g
        cons = {t.id: g.consumers(t.id) for t in g.tensors}
        src = np.transpose(self.x, (0, 2, 3, 4, 1))
        self.exact("source", self.c("source:0"), _bf(src))
        for n in g.nodes:
            if n.kind == "conv":
                xin = _t(self.c(n.inputs[0]))
                ref = _nd(F.conv3d(xin, self.w_conv(n.id), padding=1))
                self.ulp(n.id + " fwd", self.c(n.outputs[0]), ref)
            elif n.kind == "norm":
                yc = self.c(n.inputs[0])
                mean, rstd = self.stats[n.id]
                c = yc.shape[-1]
                flat = yc.reshape(-1, c)
                m64, v64 = flat.mean(0), flat.var(0)
                sd = np.sqrt(v64 + BN_EPS)
                self.n_checked += 1
                if (np.abs(mean - m64) > 1e-2 * sd).any() or \
                        (np.abs(rstd * sd - 1) > 1e-2).any():
                    self.fail.append((n.id + " stats", "mean/rstd"))
                act = cons[n.outputs[0]][0]
                gm = np.asarray(self.p[n.id + ".gamma"], np.float64)
                bt = np.asarray(self.p[n.id + ".beta"], np.float64)
                ref = np.maximum((yc - mean) * rstd * gm + bt, 0.0)
                self.ulp(n.id + " norm+relu", self.c(act + ":0"), ref, slack=1e-4)
            elif n.kind == "pool":
                a = self.c(n.inputs[0])
                ref = _nd(F.max_pool3d(_t(a), 2))
                self.exact(n.id, self.c(n.outputs[0]), ref)
            elif n.kind == "concat":
                sc, up = n.inputs
                cat = self.c(n.outputs[0])
                cs = self.c(sc).shape[-1]
                self.exact(n.id + " skip", cat[..., :cs], self.c(sc))
                upn = g.node(g.tensor(up).producer)
                xin = _t(self.c(upn.inputs[0]))
                ref = _nd(F.conv_transpose3d(xin, self.w_convt(upn.id), stride=2, padding=1,
                                             output_padding=1))
                self.ulp(upn.id + " fwd", cat[..., cs:], ref)

    # ------------------------------------------------------------------ backward
    def _dy_of(self, t):
        """The gradient tensor w.r.t. forward tensor t as the GPU stored it."""
        g = self.g
        node = g.node(g.tensor(t).producer)
        if node.kind == "upsample":
            cat = g.consumers(t)[0]
            dcat = self.c("d:" + cat + ":0")
            return dcat[..., dcat.shape[-1] // 2:]
        return self.c("d:" + t)

    def backward(self):
        g, grads = self.g, self.grads
        head = next(n for n in g.nodes if n.kind == "loss")
        for n in g.nodes:
            if n.kind == "conv":
                t_in = n.inputs[0]
                xin = _t(self.c(t_in)).requires_grad_(True)
                w = self.w_conv(n.id).requires_grad_(True)
                dy = _t(self.c("d:" + n.outputs[0]))
                F.conv3d(xin, w, padding=1).backward(dy)
                gw = w.grad.permute(0, 2, 3, 4, 1).reshape(self.p[n.id + ".w"].shape).numpy()
                self.l2(n.id + " wgrad", grads[n.id + ".w"], gw, 1e-4)
                prod = g.node(g.tensor(t_in).producer)
                if prod.kind == "source":
                    continue
                dx = _nd(xin.grad)
                if prod.kind == "activation":          # ReLU fused into the dgrad epilogue
                    if len(g.consumers(t_in)) != 1:
                        continue
                    norm = prod.inputs[0]
                    ref = dx * (self.c(t_in) > 0)
                    self.ulp(n.id + " dgrad+relu", self.c("d:" + norm), ref)
                else:                                   # pool / concat input
                    self.ulp(n.id + " dgrad", self.c("d:" + t_in), dx)
            elif n.kind == "upsample":
                t_in = n.inputs[0]
                xin = _t(self.c(t_in)).requires_grad_(True)
                w = self.w_convt(n.id).requires_grad_(True)
                dy = _t(self._dy_of(n.outputs[0]))
                F.conv_transpose3d(xin, w, stride=2, padding=1, output_padding=1).backward(dy)
                gw = w.grad.permute(1, 2, 3, 4, 0).reshape(self.p[n.id + ".w"].shape).numpy()
                self.l2(n.id + " wgrad", grads[n.id + ".w"], gw, 1e-4)
                act = g.node(g.tensor(t_in).producer)
                ref = _nd(xin.grad) * (self.c(t_in) > 0)
                self.ulp(n.id + " dgrad+relu", self.c("d:" + act.inputs[0]), ref)
            elif n.kind == "norm":
                yc = self.c(n.inputs[0])
                c = yc.shape[-1]
                mean, rstd = (v.astype(np.float64) for v in self.stats[n.id])
                dn = self.c("d:" + n.outputs[0]).reshape(-1, c)
                xhat = (yc.reshape(-1, c) - mean) * rstd
                gm = np.asarray(self.p[n.id + ".gamma"], np.float64)
                dbeta, dgamma = dn.sum(0), (dn * xhat).sum(0)
                self.l2(n.id + " dbeta", grads[n.id + ".beta"], dbeta, 1e-4)
                self.l2(n.id + " dgamma", grads[n.id + ".gamma"], dgamma, 1e-4)
                vox = dn.shape[0]
                dx = gm * rstd * (dn - dbeta / vox - xhat * dgamma / vox)
                self.l2(n.id + " bwd", self.c("d:" + n.inputs[0]).reshape(-1, c), dx, 3e-3)
            elif n.kind == "pool":
                a = self.c(n.inputs[0])
                at = _t(a).requires_grad_(True)
                F.max_pool3d(at, 2).backward(_t(self.c("d:" + n.outputs[0])))
                ref = _nd(at.grad)
                act = g.node(g.tensor(n.inputs[0]).producer)
                skip_cat = [q for q in g.consumers(n.inputs[0]) if g.node(q).kind == "concat"]
                if skip_cat:
                    dcat = self.c("d:" + skip_cat[0] + ":0")
                    ref = ref + dcat[..., :a.shape[-1]]
                ref = ref * (a > 0)
                # windows whose maximum is tied (bf16 values) may route to either voxel
                nb, d, h, w_, c = a.shape
                win = a.reshape(nb, d // 2, 2, h // 2, 2, w_ // 2, 2, c)
                mx = win.max(axis=(2, 4, 6), keepdims=True)
                tied = ((win == mx).sum(axis=(2, 4, 6), keepdims=True) > 1) & (mx > 0)
                tied = np.broadcast_to(tied, win.shape).reshape(a.shape)
                got = self.c("d:" + act.inputs[0])
                self.n_checked += 1
                err = np.abs(got - ref)
                lim = _ulp(ref) + 1e-5 * max(float(np.abs(ref).max()), 1e-30)
                bad = (err > lim) & ~tied
                if bad.any():
                    self.fail.append((n.id + " bwd+relu", "ulp", int(bad.sum())))
        # loss backward (head + softmax + soft Dice), ReLU of its input fused
        act_t = head.inputs[0]
        a = self.c(act_t)
        ncls = self.tr.cfg.n_classes
        hw = torch.as_tensor(np.asarray(self.p["head.w"], np.float64)).requires_grad_(True)
        hb = torch.as_tensor(np.asarray(self.p["head.b"], np.float64)).requires_grad_(True)
        at = _t(a).requires_grad_(True)
        logits = F.conv3d(at, hw.reshape(ncls, a.shape[-1], 1, 1, 1), hb)
        pr = torch.softmax(logits, dim=1)
        gt = F.one_hot(torch.as_tensor(self.y.astype(np.int64)), ncls).permute(0, 4, 1, 2, 3)
        gt = gt.to(torch.float64)
        inter, psum, gsum = ((pr * gt).sum(dim=(0, 2, 3, 4)), pr.sum(dim=(0, 2, 3, 4)),
                             gt.sum(dim=(0, 2, 3, 4)))
        loss = 1 - ((2 * inter + 1e-5) / (psum + gsum + 1e-5)).mean()
        loss.backward()
        self.n_checked += 1
        if abs(self.tr_loss - float(loss)) > 1e-5 * abs(float(loss)):
            self.fail.append(("loss", self.tr_loss, float(loss)))
        self.l2("head.w grad", grads["head.w"], hw.grad.numpy(), 1e-4)
        self.l2("head.b grad", grads["head.b"], hb.grad.numpy(), 1e-4)
        norm = self.g.node(self.g.tensor(act_t).producer).inputs[0]
        self.l2("loss bwd+relu", self.c("d:" + norm), _nd(at.grad) * (a > 0), 3e-3)


def check_step(tr, x, y, params, loss):
    lc = LayerCheck(tr, x, y, params)
    lc.tr_loss = loss
    lc.forward()
    lc.backward()
    return lc
