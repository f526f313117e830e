"""numpy restatement of the reference toy executor -- TEST INFRASTRUCTURE ONLY.

Follows pkg/src/swapsim/numeric.py: inputs (49-59), affine forward/backward
(62-81), residency tape (84-113), execution order (116-142), forward kinds
(201-222), loss (189-197) and grads (232-276).  Pinned bit-for-bit against
the reference's own outputs in tests/test_oracle_pinned.py.
"""
from __future__ import annotations

import zlib

import numpy as np


class OracleUseAfterSwap(Exception):
    pass


def _params(nid):
    h = zlib.crc32(nid.encode())
    return 0.7 + 0.6 * ((h & 0xFFFF) / 0xFFFF), -0.5 + ((h >> 16) / 0xFFFF)


def _count(t):
    n = t.channels
    for e in t.shape:
        n *= e
    return n


def _aff_fwd(x, n_out, a, b):
    if x.size >= n_out:
        reps = -(-x.size // n_out)
        buf = np.zeros(reps * n_out)
        buf[:x.size] = x
        return a * buf.reshape(reps, n_out).sum(axis=0) + b
    return a * np.tile(x, -(-n_out // x.size))[:n_out] + b


def _aff_bwd(dy, n_in, a):
    if n_in >= dy.size:
        return (a * np.tile(dy, -(-n_in // dy.size))[:n_in]).copy()
    reps = -(-dy.size // n_in)
    buf = np.zeros(reps * n_in)
    buf[:dy.size] = dy
    return a * buf.reshape(reps, n_in).sum(axis=0)


def _order(tg):
    g, pos = tg.graph, tg._positions
    extra: dict[int, list] = {}
    for n in g.nodes:
        if n.kind == "swap_out":
            t = n.inputs[0]
            at = max([pos[g.tensor(t).producer]] + [pos[c] for c in g.consumers(t)
                                                     if g.node(c).phase == "forward" and c in pos])
            extra.setdefault(at, []).append((0, n.id))
        elif n.kind == "swap_in":
            trig = [a for a, b in g.control_edges if b == n.id and g.node(a).kind != "swap_out"]
            extra.setdefault(max(pos[t] for t in trig), []).append((1, n.id))
    seq = []
    for p, nid in enumerate(tg.serial_order):
        seq.append(nid)
        seq.extend(x for _, x in sorted(extra.get(p, [])))
    return seq


def run_numeric(tg, plan=None, seed=0, inputs=None):
    """(loss, {input tensor: gradient}) exactly as the reference computes them."""
    g = tg.graph
    dev, host = {}, {}

    def get(t, who):
        if t not in dev:
            raise OracleUseAfterSwap(f"use-after-swap: {who} read {t}")
        return dev[t]

    for n in g.nodes:
        if n.phase == "forward" and not n.inputs and n.outputs:
            t = n.outputs[0]
            if inputs and t in inputs:
                dev[t] = np.asarray(inputs[t], dtype=np.float64).copy()
            else:
                dev[t] = np.random.default_rng((seed, zlib.crc32(n.id.encode()))) \
                    .standard_normal(_count(g.tensor(t)))
    loss_node = next((n for n in g.nodes if n.kind == "loss"), None)
    fed = set(loss_node.inputs) if loss_node else set()
    loss = 0.0
    for nid in _order(tg):
        n = g.node(nid)
        if n.kind == "swap_out":
            t = n.inputs[0]
            host[t] = get(t, nid)
            del dev[t]
        elif n.kind == "swap_in":
            out = n.outputs[0]
            src = out[:-3]
            if src not in host:
                raise OracleUseAfterSwap(f"use-after-swap: {nid} has no host copy of {src}")
            dev[out] = host[src].copy()
        elif n.kind == "loss":
            loss = 0.0
            for t in n.inputs:
                x = get(t, nid)
                loss += float(np.dot(x, x))
        elif n.kind == "grad":
            f = g.node(tg.grad_of[nid])
            inc, reuse = None, None
            for t in n.inputs:
                if g.node(g.tensor(t).producer).kind == "grad":
                    inc = get(t, nid).copy() if inc is None else inc + get(t, nid)
                else:
                    reuse = get(t, nid)
            if inc is None:
                inc = np.zeros_like(reuse)
            if f.outputs and f.outputs[0] in fed:
                inc = inc + 2.0 * reuse
            outs = n.outputs
            if not f.inputs:
                dev[outs[0]] = inc
            elif f.kind in ("conv", "matmul", "upsample", "source", "sink", "recompute"):
                dev[outs[0]] = _aff_bwd(inc, _count(g.tensor(outs[0])), _params(f.id)[0])
            elif f.kind == "activation":
                dev[outs[0]] = inc * (reuse > 0.0)
            elif f.kind == "norm":
                dev[outs[0]] = inc - inc.mean()
            elif f.kind == "pool":
                k = _count(g.tensor(outs[0])) // inc.size
                dev[outs[0]] = np.repeat(inc / k, k)[:_count(g.tensor(outs[0]))]
            elif f.kind == "concat":
                off = 0
                for o in outs:
                    sz = _count(g.tensor(o))
                    dev[o] = inc[off:off + sz].copy()
                    off += sz
        elif n.inputs:
            xs = [get(t, nid) for t in n.inputs]
            out = n.outputs[0]
            size = _count(g.tensor(out))
            kind = n.kind
            if kind in ("conv", "matmul", "upsample", "source", "sink", "recompute"):
                a, b = _params(nid.split("@rc")[0])
                dev[out] = _aff_fwd(xs[0], size, a, b)
            elif kind == "activation":
                dev[out] = np.maximum(xs[0], 0.0)
            elif kind == "norm":
                dev[out] = xs[0] - xs[0].mean()
            elif kind == "pool":
                k = xs[0].size // size
                dev[out] = xs[0][:k * size].reshape(size, k).mean(axis=1)
            elif kind == "concat":
                dev[out] = np.concatenate(xs)
    grads = {}
    for n in g.nodes:
        if n.phase == "forward" and not n.inputs and n.outputs:
            gid = f"grad/{n.id}:0"
            if g.has_tensor(gid):
                grads[n.outputs[0]] = get(gid, "<result>")
    return loss, grads
