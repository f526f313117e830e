"""Single-op entry points: run one device kernel of libunetswap on host arrays.

Used by the kernel parity tests and by bench.py's per-kernel roofline timing.
Each call builds a tiny program (upload -> op -> capture) on a shared
context; activations are NDHWC numpy arrays (float32, converted to the
requested storage dtype), weights are [Cout][27][Cin].
"""
from __future__ import annotations

import numpy as np

from ._native import ALGO_DIRECT, ALGO_IM2COL, ALGO_TCGEN05, ARENA, DT_BF16, DT_F32, OP, PERSIST, Engine
from .lowering import Program

_eng = None


def engine(arena_bytes: int = 1 << 30) -> Engine:
    global _eng
    if _eng is None or _eng.arena_bytes < arena_bytes:
        if _eng is not None:
            _eng.close()
        _eng = Engine(0, max(arena_bytes, 1 << 30))
    return _eng


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bit patterns (round to nearest even)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + 0x7FFF
    return ((u + r) >> 16).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def _store(a: np.ndarray, dtype: int) -> np.ndarray:
    return to_bf16_bits(a) if dtype == DT_BF16 else np.ascontiguousarray(a, dtype=np.float32)


def _load(raw: np.ndarray, dtype: int, shape) -> np.ndarray:
    v = from_bf16_bits(raw.view(np.uint16)) if dtype == DT_BF16 else raw.view(np.float32)
    return v.reshape(shape)


class OneOp:
    """Build and run a one-op program; inputs are staged through persistent buffers."""

    def __init__(self):
        self.pr = Program()
        self.uploads = []
        self.captures = []

    def input(self, name, arr_stored: np.ndarray, dtype: int):
        p = self.pr.tensor("<in>" + name, arr_stored.nbytes, PERSIST, dtype)
        t = self.pr.tensor(name, arr_stored.nbytes, ARENA, dtype)
        self.uploads.append((p, arr_stored))
        self.pr.op("COPY_IN", (p, t), (arr_stored.nbytes,))
        return t

    def persist(self, name, arr: np.ndarray, dtype: int):
        p = self.pr.tensor(name, arr.nbytes, PERSIST, dtype)
        self.uploads.append((p, arr))
        return p

    def output(self, name, nbytes: int, dtype: int):
        return self.pr.tensor(name, nbytes, ARENA, dtype)

    def capture(self, tid, nbytes, dtype):
        p = self.pr.tensor(f"<cap>{tid}", nbytes, PERSIST, dtype)
        self.pr.op("CAPTURE", (tid, p), (nbytes, 0))
        self.captures.append(p)
        return p

    def run(self, repeat: int = 1):
        eng = engine(self.pr.arena_need() + (64 << 20))
        self.pr.emit(eng)
        for p, arr in self.uploads:
            eng.upload(p, arr)
        for _ in range(repeat):
            eng.run()
        eng.sync()
        return eng


def last_op_seconds() -> float:
    """Device time of the op inside the last conv_op call (its slot events)."""
    tl = engine().timeline()
    return sum(e - s for node, ch, s, e in tl if ch == 0 and node == 0)


def conv_op(kind: str, x=None, w=None, dy=None, algo: int = ALGO_TCGEN05, dtype: int = DT_BF16,
            repeat: int = 1, want_stats: bool = False, relu_mask=None, x2=None):
    """kind in {conv_fwd, conv_dgrad, conv_wgrad, convt_fwd, convt_dgrad, convt_wgrad}.
    relu_mask (dgrad only): a ReLU output laid out like dx; dx is then dgrad * (mask > 0).

    Shapes: conv: x [N,D,H,W,Cin], dy [N,D,H,W,Cout]; convT: x [N,D,H,W,Cin] (low-res),
    dy [N,2D,2H,2W,Cout].  w: [Cout,27,Cin] float32.  Returns numpy float32
    (and the engine stats of the last run).

    x2 (conv_fwd / conv_wgrad, tcgen05): a second input source -- the conv reads the
    channel concatenation [x | x2] without it being materialised (dual-source concat)."""
    xa = x
    if x2 is not None:
        x = np.concatenate([x, x2], axis=-1)   # shapes only; the kernels read x and x2
    transposed = kind.startswith("convt")
    ref = x if x is not None else None
    if ref is None:
        n, d2, h2, w2, cout = dy.shape
        d, h, ww = (d2 // 2, h2 // 2, w2 // 2) if transposed else (d2, h2, w2)
        cin = w.shape[2]
    else:
        n, d, h, ww, cin = x.shape
        cout = w.shape[0] if w is not None else dy.shape[-1]
    up = 2 if transposed else 1
    vox_lo = n * d * h * ww
    vox_out = vox_lo * (8 if transposed else 1)
    o = OneOp()
    esz = 2 if dtype == DT_BF16 else 4
    grid = (n, d, h, ww)
    shape_i = [n, d, h, ww, cin, cout]
    if kind in ("conv_fwd", "convt_fwd"):
        tx = o.input("x", _store(xa if x2 is not None else x, dtype), dtype)
        tx2 = o.input("x2", _store(x2, dtype), dtype) if x2 is not None else -1
        ca = xa.shape[-1] if x2 is not None else cin
        tw = o.persist("w", _store(w, dtype), dtype)
        ty = o.output("y", vox_out * cout * esz, dtype)
        if kind == "conv_fwd":
            from ._native import workspace_bytes
            ia = shape_i + [0, algo]
            tp = o.output("part", workspace_bytes(OP["US_OP_CONV_FWD"], ia), DT_F32)
            o.pr.op("SLOT_BEGIN", (), (0, 0))
            o.pr.op("CONV_FWD", (tx, tw, ty, tp, tx2), shape_i + [0, algo, ca, 0])
            o.pr.op("SLOT_END", (), (0,))
            cp = o.capture(tp, o.pr.by_tid()[tp].nbytes, DT_F32) if want_stats else None
        else:
            o.pr.op("SLOT_BEGIN", (), (0, 0))
            o.pr.op("CONVT_FWD", (tx, tw, ty), shape_i + [0, algo])
            o.pr.op("SLOT_END", (), (0,))
            cp = None
        cy = o.capture(ty, vox_out * cout * esz, dtype)
        eng = o.run(repeat)
        out = _load(eng.download(cy, vox_out * cout * esz, np.uint8), dtype,
                    (n, d * up, h * up, ww * up, cout))
        if want_stats:
            part = eng.download(cp, o.pr.by_tid()[cp].nbytes, np.float32).reshape(-1, 2, cout)
            return out, part, eng.stats()
        return out, eng.stats()
    if kind in ("conv_dgrad", "convt_dgrad"):
        tdy = o.input("dy", _store(dy, dtype), dtype)
        tw = o.persist("w", _store(w, dtype), dtype)
        tdx = o.output("dx", vox_lo * cin * esz, dtype)
        tm = o.input("mask", _store(relu_mask, dtype), dtype) if relu_mask is not None else -1
        o.pr.op("SLOT_BEGIN", (), (0, 0))
        o.pr.op("CONV_DGRAD" if kind == "conv_dgrad" else "CONVT_DGRAD", (tdy, tw, tdx, tm),
                shape_i + [0, algo, cout, 0])
        o.pr.op("SLOT_END", (), (0,))
        cx = o.capture(tdx, vox_lo * cin * esz, dtype)
        eng = o.run(repeat)
        return _load(eng.download(cx, vox_lo * cin * esz, np.uint8), dtype,
                     (n, d, h, ww, cin)), eng.stats()
    # weight gradients
    from ._native import workspace_bytes
    tx = o.input("x", _store(xa if x2 is not None else x, dtype), dtype)
    tx2 = o.input("x2", _store(x2, dtype), dtype) if x2 is not None else -1
    tdy = o.input("dy", _store(dy, dtype), dtype)
    gbytes = cout * 27 * cin * 4
    tg = o.persist("g", np.zeros(cout * 27 * cin, np.float32), DT_F32)
    code = "CONV_WGRAD" if kind == "conv_wgrad" else "CONVT_WGRAD"
    ia = shape_i + [0, algo]
    tp = o.output("part", workspace_bytes(OP["US_OP_" + code], ia), DT_F32)
    o.pr.op("SLOT_BEGIN", (), (0, 0))
    if x2 is not None:
        o.pr.op(code, (tx, tdy, tg, tp, tx2), shape_i + [0, algo, cout, 0, xa.shape[-1]])
    else:
        o.pr.op(code, (tx, tdy, tg, tp), shape_i + [0, algo, cout, 0])
    o.pr.op("SLOT_END", (), (0,))
    eng = o.run(repeat)
    del grid
    return eng.download(tg, gbytes, np.float32).reshape(cout, 27, cin), eng.stats()


def loss_op(act, labels, hw, hb, relu: bool = False, dtype: int = DT_BF16, eps: float = 1e-5):
    """Head + soft-Dice forward and backward (LOSS_FWD then LOSS_BWD) on one batch.

    act [N,D,H,W,C] float32 (stored as dtype), labels [N,D,H,W] ints < ncls,
    hw [ncls][C], hb [ncls].  Returns (dice [3*ncls+1] float64 = per-class (I, P, G)
    sums + loss, dact float32 like act, ghw [ncls][C], ghb [ncls])."""
    from ._native import DT_F64, DT_U8, workspace_bytes
    n = act.shape[0]
    c = act.shape[-1]
    vox = int(np.prod(act.shape[1:-1]))
    ncls = hw.shape[0]
    esz = 2 if dtype == DT_BF16 else 4
    o = OneOp()
    ta = o.input("act", _store(act, dtype), dtype)
    tl = o.persist("labels", np.ascontiguousarray(labels, dtype=np.uint8).ravel(), DT_U8)
    params = np.concatenate([np.asarray(hw, np.float32).ravel(), np.asarray(hb, np.float32)])
    tp = o.persist("params", params, DT_F32)
    tdice = o.persist("dice", np.zeros(3 * ncls + 1, np.float64), DT_F64)
    tloss = o.persist("loss", np.zeros(1, np.float32), DT_F32)
    tg = o.persist("grads", np.zeros(params.size, np.float32), DT_F32)
    ia = [n, vox, c, ncls]
    tpf = o.output("partf", workspace_bytes(OP["US_OP_LOSS_FWD"], ia), DT_F32)
    tpb = o.output("partb", workspace_bytes(OP["US_OP_LOSS_BWD"], ia), DT_F32)
    tdx = o.output("dact", n * vox * c * esz, dtype)
    o.pr.op("SLOT_BEGIN", (), (0, 0))
    o.pr.op("LOSS_FWD", (ta, tl, tp, tpf, tdice, tloss), ia + [0, ncls * c], (eps,))
    o.pr.op("LOSS_BWD", (ta, tl, tp, tdice, tdx, tg, tpb),
            ia + [0, ncls * c, 0, ncls * c, 1 if relu else 0], (eps,))
    o.pr.op("SLOT_END", (), (0,))
    cx = o.capture(tdx, n * vox * c * esz, dtype)
    eng = o.run()
    dice = eng.download(tdice, (3 * ncls + 1) * 8, np.float64)
    dact = _load(eng.download(cx, n * vox * c * esz, np.uint8), dtype, act.shape)
    g = eng.download(tg, params.size * 4, np.float32)
    return dice, dact, g[:ncls * c].reshape(ncls, c), g[ncls * c:]


def stat_parts_for(shape) -> int:
    """BN partial count of a tcgen05 / im2col conv forward of this (N,D,H,W,Cin,Cout)."""
    from ._native import workspace_bytes
    n, d, h, w, cin, cout = shape
    algo = ALGO_IM2COL if cin == 4 else ALGO_TCGEN05
    return workspace_bytes(OP["US_OP_CONV_FWD"], [n, d, h, w, cin, cout, 0, algo]) // (8 * cout)


ALGOS = {"direct": ALGO_DIRECT, "tcgen05": ALGO_TCGEN05, "im2col": ALGO_IM2COL}
DTYPES = {"bf16": DT_BF16, "f32": DT_F32}
