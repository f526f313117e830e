"""Full-volume 3D U-Net training step on the B200 with planner-driven swapping.

``UNetTrainer`` is the real-op counterpart of ``run_numeric``: it builds the
reference graph (``gen_unet3d``, models.py:104), expands it
(``expand_training_graph``), applies the swap plan (``apply_rewrite`` with the
paper presets or any ``RewriteConfig``) and lowers the result to one device
program that libunetswap executes per step:

forward slots (serial positions 0..boundary)
  source      INPUT_NCDHW  (fp32 NCDHW volume -> NDHWC storage dtype)
  conv        CONV_FWD     (tcgen05 implicit GEMM, BN statistics in the epilogue)
  norm        BN_STATS + NORM_ACT (writes norm:0 *and* act:0 -- both are plan tensors)
  activation  (produced by the norm slot)
  pool        POOL_FWD ; upsample CONVT_FWD ; concat CONCAT
  loss        LOSS_FWD     (1x1x1 head + softmax + soft Dice)
backward slots -- slot grad/<f> computes the gradient of f's OUTPUT by running
the backward of f's consumers, so every slot reads exactly f:0, the tensor the
reference's reuse edge says it reads (training.py:98-130).  This makes the
planner's trigger positions (rewrite.py:177) the real prefetch deadlines:
  grad/conv  -> BN backward     grad/norm -> ReLU backward
  grad/act   -> next conv dgrad+wgrad | pool backward (+ concat shortcut) |
                transposed-conv dgrad+wgrad | loss backward
  grad/pool  -> next conv dgrad+wgrad   grad/concat -> conv dgrad+wgrad
  grad/source-> first conv wgrad        grad/upsample -> (concat split is a view)
then one optimizer slot (Adam over the flat fp32 parameters, bf16 weight copies).

Every reference tensor is materialised with exactly its planned bytes
(elem_bytes = storage bytes x batch), so swap traffic is the
plan's byte-for-byte.
"""
from __future__ import annotations

import zlib
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import (ALGO_DIRECT, ALGO_IM2COL, ALGO_TCGEN05, ARENA, CH_COMPUTE, CH_D2H, CH_H2D,
                      CH_OP, CH_STALL, DT_BF16, DT_F32, DT_F64, DT_U8, OP, PERSIST, Engine,
                      EngineError)
from .graph import GraphError
from .lowering import Program, swap_schedule
from .models import UNetParams, gen_unet3d
from .rewrite import RewriteConfig, apply_rewrite, apply_rewrites, resolve_preset
from .sim import SimReport
from .training import expand_training_graph, static_peak_estimate

BN_EPS = 1e-5
DICE_EPS = 1e-5


@dataclass
class TrainConfig:
    dims: tuple = (192, 192, 192)
    in_channels: int = 4
    base_filters: int = 64
    depth: int = 5
    convs_per_level: int = 2
    batch: int = 1
    n_classes: int = 4
    dtype: str = "bf16"              # "bf16" (tensor cores) or "f32" (check mode)
    preset: str | None = "paper-c4"  # or None with `rewrite`
    # a RewriteConfig, or a tuple of them composed left to right (rewrite.apply_rewrites:
    # recompute, then swap some of the kept checkpoints)
    rewrite: RewriteConfig | tuple | None = None
    lr: float = 5e-4                 # paper: Adam, lr 5e-4
    betas: tuple = (0.9, 0.999)
    adam_eps: float = 1e-8
    seed: int = 0
    arena_bytes: int | None = None   # HBM budget for step tensors; None = plan need + margin
    algo: str = "auto"               # "auto" | "direct"
    input_grad: bool = False         # also compute d loss / d input (not needed to train)
    capture: tuple = ()              # forward tensors to copy out (tests)
    device: int = 0
    world: int = 1                   # data-parallel ranks (gradient allreduce before Adam)
    graph: bool = True               # replay the step as a CUDA graph from the 3rd step on
    timeline: bool = True            # per-slot / per-copy timestamps (graphs need it off)
    poison: bool = False             # debug: NaN-fill every released arena region (US_FLAG_POISON)
    augment: bool = False            # random axis flips + permutations on the GPU each step
    d2h_order: str = "need"          # swap-out issue order: "need" (backward-need) or "fifo"
    dp_bucket_mb: float = 32.0       # gradient all-reduce bucket size (data parallel)
    dp_force_allreduce: bool = False  # emit the bucketed all-reduce even at world 1 (tests)
    overlap_optimizer: bool = True   # Adam per gradient bucket on the comm stream, overlapped
    # BatchNorm outputs no kernel reads (the fused NORM_ACT writes the ReLU output):
    #   "unswapped" -- not written unless the plan swaps them (planned swaps always move
    #                  their bytes: the plan runs byte for byte);
    #   "all" / True -- not written, and their planned swaps skipped (elided_swaps);
    #   "none" / False -- every BN output written
    elide_dead_norm: str | bool = "unswapped"
    direct_concat: bool = True       # convT writes its half of the concat in place
    # the concat is never materialised: the synthesis conv1 reads [skip | upsample] as two
    # sources (fprop and weight gradient), when both are device-resident where it reads them
    dual_source_concat: bool = True
    # the head's forward rides on its input's normalize pass (saves re-reading act, but the
    # per-voxel octet reduction makes the pass compute-bound: 0.35 + 0.32 -> 0.81 + 0.11 ms
    # measured r01; off by default)
    fuse_head: bool = False
    # dy's producer computes BN_BWD's channel sums (saves the sums pass, 0.31 ms per
    # full-resolution layer, but costs as much in the dgrad epilogue and more in the
    # pool / loss backward -- measured r01 a wash; off by default)
    fuse_bn_sums: bool | str = False   # True: every producer; "dgrad": conv dgrad epilogues only
                                     # with the rest of the backward
    # arena layout: "static" = planned offsets (lowering.Program.place, time-aware so a
    # swapped-out tensor's region is not reused before its D2H copy is done -- no
    # fragmentation, deterministic budgets) or "best_fit" (online allocator)
    placement: str = "static"
    slot_seconds: dict | None = None   # measured compute seconds per slot (layout timing)
    link_gbs: float = 50.0             # per-direction host-link GB/s for the layout timing

    def storage(self) -> int:
        return DT_BF16 if self.dtype == "bf16" else DT_F32

    def esz(self) -> int:
        return 2 if self.dtype == "bf16" else 4

    def unet_params(self) -> UNetParams:
        return UNetParams(dims=tuple(self.dims), in_channels=self.in_channels,
                          base_filters=self.base_filters, depth=self.depth,
                          elem_bytes=self.esz() * self.batch,
                          convs_per_level=self.convs_per_level)

    def rewrite_config(self):
        if self.rewrite is not None:
            return self.rewrite
        if self.preset:
            return resolve_preset(self.preset)
        return RewriteConfig(mode="none")


@dataclass
class ParamSlot:
    offset: int
    shape: tuple


@dataclass
class Layout:
    """Flat parameter layout (fp32 master, bf16 kernel copy, grads and Adam state)."""

    slots: dict = field(default_factory=dict)   # name -> ParamSlot
    total: int = 0

    def add(self, name: str, shape) -> int:
        n = int(np.prod(shape))
        off = self.total
        self.slots[name] = ParamSlot(off, tuple(shape))
        self.total += (n + 31) // 32 * 32      # keep every slot 128-byte aligned
        return off


def stem_supported(cin: int, cout: int, dims) -> bool:
    """The fused im2col stem kernel (csrc/conv_tc.cu, stem_geo): 4 -> 64 channels on a
    grid whose (H, W) tile into 32x4 or 16x8 voxel blocks."""
    _, h, w = dims
    return cin == 4 and cout == 64 and any(w % bw == 0 and h % (128 // bw) == 0
                                           for bw in (32, 16))


def tc_supported(kind: str, cin: int, cout: int) -> bool:
    """Shapes the tcgen05 kernels cover (csrc/conv_tc.cu); others use the direct kernels."""
    if kind in ("conv_fwd", "convt_fwd"):
        return cin % 16 == 0 and cout % 16 == 0
    if kind in ("conv_dgrad", "convt_dgrad"):
        return cin % 64 == 0 and cout % 16 == 0
    if kind == "conv_wgrad":
        return cout % 64 == 0 and (cin % 64 == 0 or (cin == 32 and cout == 64))
    if kind == "convt_wgrad":
        return cin % 64 == 0 and cout % 64 == 0 and (cin >= 128 or cout >= 128)
    raise ValueError(kind)


class UNetTrainer:
    def __init__(self, cfg: TrainConfig, device_engine: bool = True):
        self.cfg = cfg
        p = cfg.unet_params()
        self.params = p
        self.graph = gen_unet3d(p)
        self.tg = expand_training_graph(self.graph)
        self.rcfg = cfg.rewrite_config()
        if isinstance(self.rcfg, (tuple, list)):
            self.rw, self.plan = apply_rewrites(self.tg, self.rcfg)
        else:
            self.rw, self.plan = apply_rewrite(self.tg, self.rcfg)
        self.layout = Layout()
        self.bn_off: dict[str, int] = {}
        self.stat_total = 0
        self.kernel_algo: dict[str, str] = {}
        self._build_layout()
        self.program = Program()
        self.d2h_order = cfg.d2h_order
        self._lower()
        if (self.d2h_order == "need" and cfg.arena_bytes
                and self.program.order_peak() > cfg.arena_bytes):
            # deferred swap-outs keep first-level tensors allocated longer in program
            # order; under a budget that cannot hold them, keep the production order
            self.d2h_order = "fifo"
            self.layout, self.bn_off, self.stat_total, self.kernel_algo = Layout(), {}, 0, {}
            self._build_layout()
            self.program = Program()
            self._lower()
        self.liveness = static_peak_estimate(self.rw, self.plan)
        self.offsets = None
        self.layout_peak = None
        if cfg.placement == "static":
            from .engine_model import estimate_slot_seconds, plan_layout
            est = cfg.slot_seconds or estimate_slot_seconds(self.rw, dict(self.plan.clone_map))
            bw = cfg.link_gbs * 1e9
            self.offsets, self.layout_peak, self.layout_hold = plan_layout(
                self.program, est, bw, bw, cfg.arena_bytes)
            if self.offsets is None:
                # the reference's two budget failures (sim.py:33-43): one tensor larger
                # than the budget can never fit; otherwise the tensors live at the same
                # time in program order cannot be laid out in it
                from .sim import DeadlockError, InfeasibleError
                big = max((d for d in self.program.tensors.values() if d.storage == ARENA),
                          key=lambda d: d.nbytes)
                if big.nbytes > cfg.arena_bytes:
                    raise InfeasibleError(big.name, big.nbytes, cfg.arena_bytes)
                raise DeadlockError(["<arena layout>"], f"the program needs "
                                    f"{self.layout_peak} bytes at its program-order peak, "
                                    f"over the {cfg.arena_bytes}-byte budget")
            need = self.layout_peak + (64 << 20)
        else:
            need = self.program.arena_need() + (256 << 20)
        self.arena_bytes = cfg.arena_bytes if cfg.arena_bytes else need
        self.step_count = 0
        self.engine = None
        if device_engine:
            from ._native import FLAG_GRAPH, FLAG_NO_TIMELINE, FLAG_POISON
            flags = ((FLAG_GRAPH if cfg.graph else 0) | (0 if cfg.timeline else FLAG_NO_TIMELINE)
                     | (FLAG_POISON if cfg.poison else 0))
            self.engine = Engine(cfg.device, self.arena_bytes, flags)
            self.program.emit(self.engine, self.offsets)
            self._init_params()

    # ------------------------------------------------------------------ layout
    def _chan(self, tid: str) -> int:
        return self.graph.tensor(tid).channels

    def _stem(self, node) -> bool:
        """4-channel input conv run as one tcgen05 GEMM over an in-smem im2col tile."""
        cin, cout = self._chan(node.inputs[0]), self._chan(node.outputs[0])
        return (self.cfg.dtype == "bf16" and self.cfg.algo == "auto" and node.kind == "conv"
                and stem_supported(cin, cout, self.graph.tensor(node.inputs[0]).shape))

    def _conv_cin_padded(self, node) -> int:
        cin = self._chan(node.inputs[0])
        if (node.inputs[0] == "source:0" and self.cfg.dtype == "bf16" and cin % 16
                and not self._stem(node)):
            return 32   # 32-channel copy: SWIZZLE_64B operands for both fwd and wgrad
        return cin

    def _build_layout(self):
        g = self.graph
        for n in g.nodes:
            if n.kind == "conv":
                self.layout.add(n.id + ".w", (self._chan(n.outputs[0]), 27,
                                              self._conv_cin_padded(n)))
            elif n.kind == "upsample":
                self.layout.add(n.id + ".w", (self._chan(n.outputs[0]), 27,
                                              self._chan(n.inputs[0])))
            elif n.kind == "norm":
                c = self._chan(n.outputs[0])
                self.layout.add(n.id + ".gamma", (c,))
                self.layout.add(n.id + ".beta", (c,))
                self.bn_off[n.id] = self.stat_total
                self.stat_total += 2 * c
        c0 = self.cfg.base_filters
        self.layout.add("head.w", (self.cfg.n_classes, c0))
        self.layout.add("head.b", (self.cfg.n_classes,))

    def initial_params(self) -> dict:
        """Deterministic init: Kaiming-normal weights from default_rng((seed, crc32(id)))."""
        out = {}
        for name, slot in self.layout.slots.items():
            rng = np.random.default_rng((self.cfg.seed, zlib.crc32(name.encode())))
            if name.endswith(".gamma"):
                v = np.ones(slot.shape)
            elif name.endswith(".beta") or name == "head.b":
                v = np.zeros(slot.shape)
            elif name == "head.w":
                v = rng.standard_normal(slot.shape) * np.sqrt(2.0 / slot.shape[1])
            else:
                cout, _, cin = slot.shape
                node = self.graph.node(name[:-2])
                real_cin = self._chan(node.inputs[0])
                fan_in = 27 * real_cin
                v = rng.standard_normal(slot.shape) * np.sqrt(2.0 / fan_in)
                if cin != real_cin:
                    v[:, :, real_cin:] = 0.0
            out[name] = v.astype(np.float32)
        return out

    def _flat(self, named: dict) -> np.ndarray:
        flat = np.zeros(self.layout.total, np.float32)
        for name, slot in self.layout.slots.items():
            n = int(np.prod(slot.shape))
            flat[slot.offset:slot.offset + n] = np.asarray(named[name], np.float32).reshape(-1)
        return flat

    def unflat(self, flat: np.ndarray) -> dict:
        out = {}
        for name, slot in self.layout.slots.items():
            n = int(np.prod(slot.shape))
            out[name] = flat[slot.offset:slot.offset + n].reshape(slot.shape).copy()
        return out

    def _init_params(self):
        flat = self._flat(self.initial_params())
        e = self.engine
        e.upload(self.t_P, flat)
        if self.cfg.dtype == "bf16":
            from .ops import to_bf16_bits
            e.upload(self.t_PB, to_bf16_bits(flat))
        e.sync()

    # ------------------------------------------------------------------ lowering
    def _lower(self):
        cfg, g, pr = self.cfg, self.rw.graph, self.program
        dt, esz, N = cfg.storage(), cfg.esz(), cfg.batch
        fwd_graph = self.graph
        P = self.layout.total
        self.t_P = pr.tensor("<params>", P * 4, PERSIST, DT_F32)
        self.t_G = pr.tensor("<grads>", P * 4, PERSIST, DT_F32)
        self.t_M = pr.tensor("<adam.m>", P * 4, PERSIST, DT_F32)
        self.t_V = pr.tensor("<adam.v>", P * 4, PERSIST, DT_F32)
        self.t_PB = pr.tensor("<params.bf16>", P * 2, PERSIST, DT_BF16)
        self.t_STAT = pr.tensor("<bn.stats>", max(1, self.stat_total) * 4, PERSIST, DT_F32)
        ncls = cfg.n_classes
        self.t_DICE = pr.tensor("<dice>", (3 * ncls + 1) * 8, PERSIST, DT_F64)
        self.t_LOSS = pr.tensor("<loss>", 4, PERSIST, DT_F32)
        D, H, W = cfg.dims
        vox0 = D * H * W
        self.t_IN = pr.tensor("<input>", N * cfg.in_channels * vox0 * 4, PERSIST, DT_F32)
        self.t_LBL = pr.tensor("<labels>", N * vox0, PERSIST, DT_U8)
        # augmentation: the flipped / permuted labels the loss reads (written every step)
        self.t_labels = (pr.tensor("<labels.aug>", N * vox0, PERSIST, DT_U8) if cfg.augment
                         else self.t_LBL)
        wts = self.t_PB if cfg.dtype == "bf16" else self.t_P
        self.captured = {}
        for t in cfg.capture:
            tt = fwd_graph.tensor(t[2:] if t.startswith("d:") else t)
            nb = N * int(np.prod(tt.shape)) * tt.channels * esz
            self.captured[t] = pr.tensor("<capture>" + t, nb, PERSIST, dt)

        # every graph tensor and every gradient-of-output tensor, at real bytes
        def shape_of(t):
            tt = fwd_graph.tensor(t)
            return tt.shape, tt.channels

        for t in g.tensors:
            if g.node(t.producer).kind == "grad":
                continue
            # "<t>@in" (swap-in copy) and "<t>@rc<s>" (recompute clone) have t's shape
            shp, c = shape_of(t.id.split("@")[0])
            nbytes = N * int(np.prod(shp)) * c * esz
            pr.tensor(t.id, nbytes, ARENA, dt)
        for t in fwd_graph.tensors:
            shp, c = t.shape, t.channels
            pr.tensor("d:" + t.id, N * int(np.prod(shp)) * c * esz, ARENA, dt)

        sched = swap_schedule(self.rw, self.plan)
        swapped = sched.swapped
        T = pr.tid
        d2h_slot = self._d2h_issue_slots(swapped, {t: pr.tensors[t].nbytes for t in swapped})
        deferred = {}    # slot -> swap-outs issued after it, in issue order
        for t, e in sorted(d2h_slot.items(), key=lambda kv: kv[1][1]):
            if e[0] != self.rw.position(self.rw.graph.tensor(t).producer):
                deferred.setdefault(e[0], []).append(t)
        release_at = {}
        for p0, ts in sched.release_after.items():
            for t in ts:   # a deferred swap-out moves its release behind it
                release_at.setdefault(max(p0, d2h_slot[t][0]), []).append(t)

        def fwd_t(t):        # forward-phase name of a tensor
            return t

        clone_of = dict(self.plan.clone_map) if self.plan is not None else {}
        alias = {}           # within a grad slot: forward tensor -> the copy it reads

        def bwd_t(t):        # backward readers go through the prefetched / recomputed copy
            if t in alias:
                return alias[t]
            return t + "@in" if t in swapped else t

        def grid(t):
            tt = fwd_graph.tensor(t)
            return tt.shape

        def algo_for(kind, cin, cout, name, dims=None):
            if (cfg.dtype == "bf16" and cfg.algo == "auto" and kind in ("conv_fwd", "conv_wgrad")
                    and dims is not None and stem_supported(cin, cout, dims)):
                self.kernel_algo[name] = "im2col-tcgen05"
                return ALGO_IM2COL
            a = ALGO_TCGEN05 if (cfg.dtype == "bf16" and cfg.algo == "auto"
                                 and tc_supported(kind, cin, cout)) else ALGO_DIRECT
            self.kernel_algo[name] = "tcgen05" if a == ALGO_TCGEN05 else "direct"
            return a

        def stat_parts(ia):
            """BN partial count a CONV_FWD writes (its workspace is exactly the partials)."""
            return ws("CONV_FWD", ia) // (8 * ia[5])

        io_counter = [0]
        consumers = {t.id: [c for c in fwd_graph.consumers(t.id)] for t in fwd_graph.tensors}
        # upsample outputs written straight into their concat (channel slice [C, 2C)): the
        # concat then copies only the skip half.  Needs the tcgen05 convT, and the upsample
        # output must be an ordinary tensor -- not swapped, captured or recomputed.
        self.direct_up = {}
        for n in fwd_graph.nodes:
            if n.kind != "upsample" or not cfg.direct_concat or cfg.dtype != "bf16":
                continue
            up = n.outputs[0]
            cons = consumers[up]
            if len(cons) != 1 or fwd_graph.node(cons[0]).kind != "concat":
                continue
            cat = fwd_graph.node(cons[0])
            if cat.inputs[1] != up or up in swapped or up in self.captured:
                continue
            if n.id in clone_of.values() or cat.id in clone_of.values():
                continue
            if any(k.split("@")[0] in (n.id, cat.id) for k in clone_of):
                continue
            cin, cout = self._chan(n.inputs[0]), self._chan(up)
            if not tc_supported("convt_fwd", cin, cout) or cfg.algo != "auto":
                continue
            self.direct_up[up] = cat.outputs[0]
        # dual-source concats: {concat tensor: (skip, upsample)} -- never written; the conv
        # that reads the concat takes its two halves as separate TMA sources.  Requires a
        # concat nobody swaps or captures, halves nobody swaps (the skip must stay resident
        # from the forward conv through the backward weight gradient), 64-channel multiples
        # and the tcgen05 fprop / wgrad.
        self.dual_cat = {}
        for n in fwd_graph.nodes:
            if n.kind != "concat" or not cfg.dual_source_concat or cfg.dtype != "bf16":
                continue
            a, b = n.inputs
            cat = n.outputs[0]
            cons = consumers[cat]
            if len(cons) != 1 or fwd_graph.node(cons[0]).kind != "conv":
                continue
            conv = fwd_graph.node(cons[0])
            ca, cb = self._chan(a), self._chan(b)
            cout = self._chan(conv.outputs[0])
            if ca % 64 or cb % 64 or cfg.algo != "auto":
                continue
            if any(t in swapped or t in self.captured for t in (a, b, cat)):
                continue
            if self.plan is not None and cat in self.plan.checkpoints:
                continue   # a kept checkpoint is read as one tensor by a recompute clone
            if not (tc_supported("conv_fwd", ca + cb, cout)
                    and tc_supported("conv_wgrad", ca + cb, cout)):
                continue
            self.dual_cat[cat] = (a, b)
            self.direct_up.pop(b, None)
        loss_node = next(n for n in fwd_graph.nodes if n.kind == "loss")
        src_pad = {}  # name of the padded source copy per phase

        def ws(opname, iargs):
            return _native.workspace_bytes(OP["US_OP_" + opname], iargs)

        scratch_id = [0]

        def scratch(tag, nbytes, dtype=DT_F32):
            scratch_id[0] += 1
            return pr.tensor(f"<{tag}#{scratch_id[0]}>", max(16, nbytes), ARENA, dtype)

        def conv_input(node, phase, xin=None):
            """Tensor id (program) feeding a conv; pads the 4-channel source for tcgen05."""
            x = node.inputs[0]
            if xin is None:
                xin = fwd_t(x) if phase == "fwd" else bwd_t(x)
            cin_pad = self._conv_cin_padded(node)
            if cin_pad == self._chan(x):
                return T(xin), cin_pad
            key = (x, phase)
            if key not in src_pad:
                dd, hh, ww = grid(x)
                tp = pr.tensor(f"<pad:{x}:{phase}>", N * dd * hh * ww * cin_pad * esz, ARENA, dt)
                pr.op("PAD_CH", (T(xin), tp), (N * dd * hh * ww, self._chan(x), cin_pad))
                src_pad[key] = tp
            return src_pad[key], cin_pad

        parts = {}  # conv node -> stats partial tensor

        def lower_forward(n):
            if n.kind == "source":
                out = n.outputs[0]
                if cfg.augment:   # random flips / permutation, drawn per step (run_async)
                    pr.op("INPUT_NCDHW", (self.t_IN, T(out)),
                          (N, cfg.in_channels, D, H, W, cfg.in_channels), (0, 0))
                    pr.op("LABELS_AUG", (self.t_LBL, self.t_labels), (N, D, H, W), (0, 0))
                else:
                    pr.op("INPUT_NCDHW", (self.t_IN, T(out)), (N, cfg.in_channels, D, H, W,
                                                              cfg.in_channels))
            elif n.kind == "conv":
                tx, cin = conv_input(n, "fwd")
                cout = self._chan(n.outputs[0])
                dd, hh, ww = grid(n.outputs[0])
                algo = algo_for("conv_fwd", cin, cout, n.id + ".fwd", (dd, hh, ww))
                ia = [N, dd, hh, ww, cin, cout, self.layout.slots[n.id + ".w"].offset, algo]
                tp = scratch("bnpart", ws("CONV_FWD", ia))
                parts[n.id] = (tp, stat_parts(ia))
                if n.inputs[0] in self.dual_cat:   # [skip | upsample] as two sources
                    sa, sb = self.dual_cat[n.inputs[0]]
                    pr.op("CONV_FWD", (T(sa), wts, T(n.outputs[0]), tp, T(sb)),
                          ia + [self._chan(sa), 0])
                else:
                    pr.op("CONV_FWD", (tx, wts, T(n.outputs[0]), tp), ia + [cin, 0])
            elif n.kind == "norm":
                conv = n.inputs[0]
                cnode = fwd_graph.tensor(conv).producer
                c = self._chan(conv)
                dd, hh, ww = grid(conv)
                vox = N * dd * hh * ww
                tp, nparts = parts[cnode]
                pr.op("BN_STATS", (tp, self.t_STAT), (nparts, c, vox, self.bn_off[n.id]),
                      (BN_EPS,))
                act = consumers[n.outputs[0]][0]
                act_t = act + ":0"
                ia_na = [vox, c, self.bn_off[n.id], self.layout.slots[n.id + ".gamma"].offset,
                         self.layout.slots[n.id + ".beta"].offset]
                head = [fwd_graph.node(q) for q in consumers.get(act_t, [])]
                if (cfg.fuse_head and cfg.dtype == "bf16" and c == 64 and 2 <= ncls <= 8
                        and len(head) == 1 and head[0].kind == "loss"
                        and act_t not in swapped and act_t not in self.captured):
                    # the head forward rides on the normalize pass: its Dice partials go to
                    # the loss slot's LOSS_FWD, which then only finalizes them
                    tpl = scratch("losspart", ws("LOSS_FWD", [N, vox // N, c, ncls]))
                    self._loss_pre = tpl
                    pr.op("NORM_ACT", (T(conv), self.t_STAT, self.t_P, T(n.outputs[0]),
                                       T(act_t), self.t_labels, tpl),
                          ia_na + [ncls, self.layout.slots["head.w"].offset,
                                   self.layout.slots["head.b"].offset])
                else:
                    pr.op("NORM_ACT", (T(conv), self.t_STAT, self.t_P, T(n.outputs[0]),
                                       T(act_t)), ia_na)
            elif n.kind == "activation":
                pass   # written by the preceding norm slot (fused apply)
            elif n.kind == "pool":
                x = n.inputs[0]
                dd, hh, ww = grid(x)
                pr.op("POOL_FWD", (T(x), T(n.outputs[0])), (N, dd, hh, ww, self._chan(x)))
            elif n.kind == "upsample":
                x = n.inputs[0]
                dd, hh, ww = grid(x)
                cin, cout = self._chan(x), self._chan(n.outputs[0])
                algo = algo_for("convt_fwd", cin, cout, n.id + ".fwd")
                ia = [N, dd, hh, ww, cin, cout, self.layout.slots[n.id + ".w"].offset, algo]
                cat_out = self.direct_up.get(n.outputs[0])
                if cat_out is not None:   # into y[:, C:2C] of the concat
                    pr.op("CONVT_FWD", (T(x), wts, T(cat_out)), ia + [2 * cout, cout])
                else:
                    pr.op("CONVT_FWD", (T(x), wts, T(n.outputs[0])), ia)
            elif n.kind == "concat":
                a, b = n.inputs
                if n.outputs[0] in self.dual_cat:
                    return   # read in place by its conv (two sources)
                dd, hh, ww = grid(a)
                ia = [N * dd * hh * ww, self._chan(a), self._chan(b)]
                if b in self.direct_up:
                    pr.op("CONCAT", (T(a), -1, T(n.outputs[0])), ia + [1])
                else:
                    pr.op("CONCAT", (T(a), T(b), T(n.outputs[0])), ia)
            elif n.kind == "loss":
                x = n.inputs[0]
                dd, hh, ww = grid(x)
                vox = dd * hh * ww
                c = self._chan(x)
                ia = [N, vox, c, ncls]
                pre = getattr(self, "_loss_pre", None)
                self._loss_pre = None
                tp = pre if pre is not None else scratch("losspart", ws("LOSS_FWD", ia))
                pr.op("LOSS_FWD", (T(x), self.t_labels, self.t_P, tp, self.t_DICE, self.t_LOSS),
                      ia + [self.layout.slots["head.w"].offset,
                            self.layout.slots["head.b"].offset, 1 if pre is not None else 0],
                      (DICE_EPS,))
            else:
                raise GraphError(f"engine has no kernel for node kind {n.kind!r}")

        relu_fused = set()   # activations whose backward ran inside their gradient's producer

        def fuse_relu(f, tensor_core=True):
            """Fuse ReLU backward into the op producing d:act (dgrad / pool / loss epilogue):
            it then writes d:norm = d:act * (act > 0) and the grad/norm slot only touches
            norm:0.  bf16 only (the fp32 check mode keeps the separate RELU_BWD)."""
            return f.kind == "activation" and cfg.dtype == "bf16" and tensor_core

        def grad_target(f, fused):
            """(tensor written, mask operand) for the gradient of f's output."""
            if fused:
                relu_fused.add(f.id)
                return T("d:" + f.inputs[0]), True
            return T("d:" + f.outputs[0]), False

        bn_pre = {}   # norm node -> partials tensor its dy's producer writes (BN_BWD skips them)

        def bn_operands(f, fused, producer="dgrad"):
            """Extra (tensors, iargs) for the op producing d:norm, so it folds BN_BWD's
            (sum dy, sum dy * xhat) pass into its epilogue: the BN input, the statistics and
            a partials tensor.  Only when the BN input is plainly resident (not swapped or
            recomputed: the producer runs a slot before BN_BWD, ahead of its prefetch)."""
            if not fused or not cfg.fuse_bn_sums:
                return (), ()
            if cfg.fuse_bn_sums == "dgrad" and producer != "dgrad":
                return (), ()
            norm = fwd_graph.node(fwd_graph.tensor(f.inputs[0]).producer)
            if norm.kind != "norm":
                return (), ()
            xin = norm.inputs[0]
            conv = fwd_graph.tensor(xin).producer
            if xin in swapped or xin in alias or conv in clone_of.values():
                return (), ()
            c = self._chan(xin)
            dd, hh, ww = grid(xin)
            tp = scratch("bnpre", ws("BN_BWD", [N * dd * hh * ww, c]))
            bn_pre[norm.id] = tp
            return (T(xin), self.t_STAT, tp), (self.bn_off[norm.id],)

        def consumer_backward(f, c, out_t):
            """Backward of consumer c w.r.t. its input f:0; writes/accumulates d:f:0 (or
            d:norm:0 when f is a ReLU fused into this op).
            Returns True if it wrote the gradient itself."""
            x = f.outputs[0]
            dx = T("d:" + x)
            cn = fwd_graph.node(c)
            if cn.kind == "conv":
                tx, cin = conv_input(cn, "bwd")
                cout = self._chan(cn.outputs[0])
                dd, hh, ww = grid(x)
                woff = self.layout.slots[cn.id + ".w"].offset
                need_dx = f.kind != "source" or cfg.input_grad
                if need_dx:
                    algo = algo_for("conv_dgrad", cin, cout, cn.id + ".dgrad")
                    if cin != self._chan(x):
                        raise GraphError("input gradient through a padded conv is not supported")
                    dx, fused = grad_target(f, fuse_relu(f, algo == ALGO_TCGEN05))
                    bt, bi = bn_operands(f, fused)
                    pr.op("CONV_DGRAD", (T("d:" + cn.outputs[0]), wts, dx,
                                         T(out_t) if fused else -1) + bt,
                          (N, dd, hh, ww, cin, cout, woff, algo, cout, 0) + bi)
                walgo = algo_for("conv_wgrad", cin, cout, cn.id + ".wgrad", (dd, hh, ww))
                ia = [N, dd, hh, ww, cin, cout, woff, walgo]
                tp = scratch("wgpart", ws("CONV_WGRAD", ia))
                if x in self.dual_cat:   # the halves this slot's concat copy is made of
                    sa, sb = self.dual_cat[x]
                    ver = alias.get(x)
                    if ver is not None:  # a recompute clone: read the clone's inputs
                        sa, sb = self.rw.graph.node(self.rw.graph.tensor(ver).producer).inputs
                    pr.op("CONV_WGRAD", (T(sa), T("d:" + cn.outputs[0]), self.t_G, tp, T(sb)),
                          ia + [cout, 0, self._chan(self.dual_cat[x][0])])
                else:
                    pr.op("CONV_WGRAD", (tx, T("d:" + cn.outputs[0]), self.t_G, tp),
                          ia + [cout, 0])
                return need_dx
            if cn.kind == "norm":
                cx = self._chan(x)
                dd, hh, ww = grid(x)
                vox = N * dd * hh * ww
                ia = [vox, cx]
                pre = bn_pre.pop(cn.id, None)
                tp = pre if pre is not None else scratch("bnbwd", ws("BN_BWD", ia))
                pr.op("BN_BWD", (T(out_t), T("d:" + cn.outputs[0]), self.t_STAT, self.t_P,
                                 self.t_G, dx, tp),
                      (vox, cx, self.bn_off[cn.id], self.layout.slots[cn.id + ".gamma"].offset,
                       self.layout.slots[cn.id + ".gamma"].offset,
                       self.layout.slots[cn.id + ".beta"].offset, 1 if pre is not None else 0))
                return True
            if cn.kind == "activation":
                if cn.id in relu_fused:   # already applied by d:act's producer
                    return False
                dd, hh, ww = grid(x)
                pr.op("RELU_BWD", (T("d:" + cn.outputs[0]), T(out_t), dx),
                      (N * dd * hh * ww * self._chan(x),))
                return True
            if cn.kind == "upsample":
                dd, hh, ww = grid(x)
                cin, cout = self._chan(x), self._chan(cn.outputs[0])
                woff = self.layout.slots[cn.id + ".w"].offset
                # d:upsample:0 is the [C:2C] channel slice of d:concat:0
                cat = consumers[cn.outputs[0]][0]
                dy_t = T("d:" + cat + ":0")
                algo = algo_for("convt_dgrad", cin, cout, cn.id + ".dgrad")
                dx, fused = grad_target(f, fuse_relu(f, algo == ALGO_TCGEN05))
                bt, bi = bn_operands(f, fused)
                pr.op("CONVT_DGRAD", (dy_t, wts, dx, T(out_t) if fused else -1) + bt,
                      (N, dd, hh, ww, cin, cout, woff, algo, 2 * cout, cout) + bi)
                walgo = algo_for("convt_wgrad", cin, cout, cn.id + ".wgrad")
                ia = [N, dd, hh, ww, cin, cout, woff, walgo]
                tp = scratch("wgpart", ws("CONVT_WGRAD", ia))
                pr.op("CONVT_WGRAD", (T(out_t), dy_t, self.t_G, tp), ia + [2 * cout, cout])
                return True
            if cn.kind == "loss":
                dd, hh, ww = grid(x)
                c = self._chan(x)
                ia = [N, dd * hh * ww, c, ncls]
                tp = scratch("lossbwd", ws("LOSS_BWD", ia))
                dx, fused = grad_target(f, fuse_relu(f))
                bt, bi = bn_operands(f, fused, "loss")
                pr.op("LOSS_BWD", (T(out_t), self.t_labels, self.t_P, self.t_DICE, dx, self.t_G,
                                   tp) + bt,
                      ia + [self.layout.slots["head.w"].offset, self.layout.slots["head.b"].offset,
                            self.layout.slots["head.w"].offset, self.layout.slots["head.b"].offset,
                            1 if fused else 0] + list(bi),
                      (DICE_EPS,))
                return True
            raise GraphError(f"no backward for consumer kind {cn.kind!r}")

        def lower_clone(cn):
            """Recompute clone ``<f>@rc<s>`` (reference insert_recompute, rewrite.py:237-353):
            the forward op again, reading kept tensors or earlier clones.  BN reuses the
            statistics saved by the forward pass, so the clone is bit-identical to f:0."""
            f = fwd_graph.node(clone_of[cn.id])
            out, ins = cn.outputs[0], cn.inputs
            base = f.outputs[0]
            if f.kind == "conv":
                tx, cin = conv_input(f, "rc:" + out, xin=ins[0])
                cout = self._chan(base)
                dd, hh, ww = grid(base)
                # same kernel as the original (the 4-channel stem included: without the
                # grid a stem clone fell back to the CUDA-core direct conv, 58 ms at 192^3)
                algo = algo_for("conv_fwd", cin, cout, f.id + ".fwd", (dd, hh, ww))
                ia = [N, dd, hh, ww, cin, cout, self.layout.slots[f.id + ".w"].offset, algo]
                tp = scratch("bnpart", ws("CONV_FWD", ia))
                if f.inputs[0] in self.dual_cat:   # reads the (skipped) concat clone's inputs
                    sa, sb = self.rw.graph.node(self.rw.graph.tensor(ins[0]).producer).inputs
                    pr.op("CONV_FWD", (T(sa), wts, T(out), tp, T(sb)),
                          ia + [self._chan(self.dual_cat[f.inputs[0]][0]), 0])
                else:
                    pr.op("CONV_FWD", (tx, wts, T(out), tp), ia + [cin, 0])
            elif f.kind == "norm":
                c = self._chan(base)
                dd, hh, ww = grid(base)
                pr.op("NORM_ACT", (T(ins[0]), self.t_STAT, self.t_P, T(out), -1),
                      (N * dd * hh * ww, c, self.bn_off[f.id],
                       self.layout.slots[f.id + ".gamma"].offset,
                       self.layout.slots[f.id + ".beta"].offset))
            elif f.kind == "activation":
                dd, hh, ww = grid(base)
                pr.op("RELU_FWD", (T(ins[0]), T(out)), (N * dd * hh * ww * self._chan(base),))
            elif f.kind == "pool":
                x = f.inputs[0]
                dd, hh, ww = grid(x)
                pr.op("POOL_FWD", (T(ins[0]), T(out)), (N, dd, hh, ww, self._chan(x)))
            elif f.kind == "upsample":
                x = f.inputs[0]
                dd, hh, ww = grid(x)
                cin, cout = self._chan(x), self._chan(base)
                algo = algo_for("convt_fwd", cin, cout, f.id + ".fwd")
                pr.op("CONVT_FWD", (T(ins[0]), wts, T(out)),
                      (N, dd, hh, ww, cin, cout, self.layout.slots[f.id + ".w"].offset, algo))
            elif f.kind == "concat":
                if base in self.dual_cat:
                    return   # the weight gradient reads the clone's two inputs directly
                a = f.inputs[0]
                dd, hh, ww = grid(a)
                pr.op("CONCAT", (T(ins[0]), T(ins[1]), T(out)),
                      (N * dd * hh * ww, self._chan(a), self._chan(f.inputs[1])))
            else:
                raise GraphError(f"engine cannot recompute node kind {f.kind!r}")

        def lower_grad(gnode):
            # the grad slot reads f:0 through whatever copy the plan rewired it to
            alias.clear()
            for t in gnode.inputs:
                if "@" in t:
                    alias[t.split("@")[0]] = t
            f = fwd_graph.node(self.rw.grad_of[gnode.id])
            if f.kind == "loss":
                return
            x = f.outputs[0]
            xin = bwd_t(x)
            cons = consumers[x]
            kinds = sorted(fwd_graph.node(c).kind for c in cons)
            if kinds == ["concat", "pool"]:
                pool = next(c for c in cons if fwd_graph.node(c).kind == "pool")
                cat = next(c for c in cons if fwd_graph.node(c).kind == "concat")
                dd, hh, ww = grid(x)
                c = self._chan(x)
                dx, fused = grad_target(f, fuse_relu(f))
                bt, bi = bn_operands(f, fused, "pool")
                pr.op("POOL_BWD", (T(xin), T("d:" + pool + ":0"), T("d:" + cat + ":0"), dx) + bt,
                      (N, dd, hh, ww, c, 2 * c, 0, 1 if fused else 0) + bi)
            elif kinds == ["pool"]:
                pool = cons[0]
                dd, hh, ww = grid(x)
                c = self._chan(x)
                dx, fused = grad_target(f, fuse_relu(f))
                bt, bi = bn_operands(f, fused, "pool")
                pr.op("POOL_BWD", (T(xin), T("d:" + pool + ":0"), -1, dx) + bt,
                      (N, dd, hh, ww, c, 0, 0, 1 if fused else 0) + bi)
            elif kinds == ["concat"]:
                if x not in self.direct_up:   # (a direct upsample output never existed)
                    pr.op("TOUCH", (T(xin),))   # concat split is a view; the slot still owns x
            elif len(cons) == 1:
                wrote = consumer_backward(f, cons[0], xin)
                if not wrote:
                    pr.op("TOUCH", (T(xin),))
            else:
                raise GraphError(f"unsupported consumer pattern {kinds} for {x!r}")

        # ---- emit slots
        for p, nid in enumerate(self.rw.serial_order):
            n = g.node(nid)
            pr.slot_names[p] = nid
            pr.slot_phase[p] = n.phase
            pr.op("SLOT_BEGIN", (), (p, 0 if n.phase == "forward" else 1))
            if n.kind == "grad":
                lower_grad(n)
                alias.clear()
            elif nid in clone_of:
                lower_clone(n)
            else:
                lower_forward(fwd_graph.node(nid))
                for t in n.outputs:
                    if t in self.captured:
                        pr.op("CAPTURE", (T(t), self.captured[t]),
                              (pr.tensors[t].nbytes, 0))
            def swap_out(t):
                io = io_counter[0]
                io_counter[0] += 1
                pr.io_names[io] = swapped[t][0]
                pr.op("SWAP_OUT", (T(t),), (io,))

            if n.kind == "norm" and nid not in clone_of:
                act = consumers[n.outputs[0]][0] + ":0"
                if act in self.captured:
                    pr.op("CAPTURE", (T(act), self.captured[act]), (pr.tensors[act].nbytes, 0))
            pr.op("SLOT_END", (), (p,))
            # swap-outs are ready when the producer slot ends (sim.py:229-236)
            for t in n.outputs:
                if t in swapped and d2h_slot[t][0] == p:
                    swap_out(t)
            for t in deferred.get(p, ()):
                swap_out(t)
            for t in sorted(release_at.get(p, ())):
                pr.op("SWAP_RELEASE", (T(t),))
            for src, in_node in sched.prefetch_after.get(p, ()):
                io = io_counter[0]
                io_counter[0] += 1
                pr.io_names[io] = in_node
                pr.op("SWAP_IN", (T(src), T(src + "@in")), (io, p))
        # optimizer slot
        opt = len(self.rw.serial_order)
        pr.slot_names[opt] = "optimizer"
        pr.slot_phase[opt] = "optimizer"
        pr.op("SLOT_BEGIN", (), (opt, 2))
        if not (cfg.overlap_optimizer or cfg.world > 1 or cfg.dp_force_allreduce):
            pr.op("ADAM", (self.t_P, self.t_G, self.t_M, self.t_V, self.t_PB),
                  (self.layout.total, 1 if cfg.dtype == "bf16" else 0),
                  (cfg.lr, cfg.betas[0], cfg.betas[1], cfg.adam_eps, 1.0))
        pr.op("SLOT_END", (), (opt,))
        if cfg.overlap_optimizer or cfg.world > 1 or cfg.dp_force_allreduce:
            self._insert_grad_buckets()
        self.dead_norm_outputs = []
        self.elided_swaps = []
        mode = {True: "all", False: "none"}.get(cfg.elide_dead_norm, cfg.elide_dead_norm)
        if mode not in ("unswapped", "all", "none"):
            raise GraphError(f"elide_dead_norm must be 'unswapped', 'all' or 'none', not {mode!r}")
        if mode != "none":
            self._drop_dead_norm_outputs(keep_swapped=mode == "unswapped")
        self._capture_gradients()
        pr.insert_frees()
        self._adam_engine_index = [k for k, op in enumerate(pr.ops)
                                   if op[0] == OP["US_OP_ADAM"]]

    # operand position of the gradient an op writes (opcodes.h)
    _GRAD_OUT = {"BN_BWD": 5, "RELU_BWD": 2, "CONV_DGRAD": 2, "CONVT_DGRAD": 2, "POOL_BWD": 3,
                 "LOSS_BWD": 4}

    def _capture_gradients(self):
        """Tests: copy requested activation gradients ("d:<tensor>") out right after the
        last op that writes them (a ReLU gradient fused into its producer is never
        materialised: request the BN output's gradient instead)."""
        pr = self.program
        want = [t for t in self.captured if t.startswith("d:")]
        if not want:
            return
        out_pos = {OP["US_OP_" + k]: v for k, v in self._GRAD_OUT.items()}
        inserts = []
        for t in want:
            tid = pr.tid(t)
            last = max((k for k, (code, tids, _, _) in enumerate(pr.ops)
                        if code in out_pos and len(tids) > out_pos[code]
                        and tids[out_pos[code]] == tid), default=None)
            if last is None:
                raise GraphError(f"no op writes {t!r} (fused into its producer?)")
            inserts.append((last, (OP["US_OP_CAPTURE"], (tid, self.captured[t]),
                                   (pr.tensors[t].nbytes, 0), ())))
        for k, op in sorted(inserts, key=lambda kv: -kv[0]):
            pr.ops.insert(k + 1, op)

    def _drop_dead_norm_outputs(self, keep_swapped: bool = False):
        """NORM_ACT writes the BatchNorm output only if a later kernel reads it.

        The graph keeps norm and ReLU as separate nodes (models.py:62-75), but the fused
        NORM_ACT produces the ReLU output directly, the BN backward reads the conv
        output and the ReLU backward the ReLU output.  The norm tensor is therefore dead
        unless a recompute clone reads it.  A dead one is neither written (906 MB per
        full-resolution layer) nor allocated, and its bookkeeping reads go with it: the
        grad slot's TOUCH (a residency read) and, when the plan swaps it, its swap-out,
        release and prefetch -- moving bytes no kernel will read.  The plan itself is
        unchanged (parity); `elided_swaps` lists the planned swaps not executed."""
        pr = self.program
        bookkeeping = {OP["US_OP_TOUCH"], OP["US_OP_SWAP_OUT"], OP["US_OP_SWAP_IN"],
                       OP["US_OP_SWAP_RELEASE"]}
        uses: dict[int, int] = {}
        swap_in_of: dict[int, int] = {}
        for code, tids, _, _ in pr.ops:
            if code == OP["US_OP_SWAP_IN"]:
                swap_in_of[tids[0]] = tids[1]
            if code in bookkeeping:
                continue
            for t in tids:
                if t >= 0:
                    uses[t] = uses.get(t, 0) + 1
        na = OP["US_OP_NORM_ACT"]
        dead = set()
        for k, (code, tids, ia, fa) in enumerate(pr.ops):
            if code != na or tids[3] < 0 or tids[4] < 0 or uses[tids[3]] != 1:
                continue
            t_in = swap_in_of.get(tids[3])
            if t_in is not None and (keep_swapped or uses.get(t_in, 0)):
                continue
            dead.add(tids[3])
            if t_in is not None:
                dead.add(t_in)
            pr.ops[k] = (code, tids[:3] + (-1,) + tids[4:], ia, fa)
        pr.ops = [op for op in pr.ops
                  if not (op[0] in bookkeeping and any(t in dead for t in op[1]))]
        defs = pr.by_tid()
        self.dead_norm_outputs = sorted(dead)
        self.elided_swaps = sorted(defs[t].name for t in dead if t in swap_in_of)

    def _d2h_issue_slots(self, swapped: dict, nbytes: dict) -> dict:
        """Where each swap-out is issued: tensor -> (slot, rank in the D2H FIFO).

        The copy engine serves D2H copies in issue order, and on the B200 the forward
        produces every swapped tensor long before the link has moved them (7.47 GB at
        ~55 GB/s for paper-c4 vs a ~25 ms forward).  Issued at production ("fifo", the
        reference simulator's order, sim.py:229-236), the first-level tensors occupy the
        link while the deep tensors the backward needs FIRST wait behind them, and no
        prefetch can start before the whole D2H queue drains.  "need" issues them in
        backward-need order instead: a list schedule over estimated slot times (the
        reference cost model, models.py:14-39, at B200 rates) picks, whenever the link
        frees up, the produced tensor whose first backward reader comes earliest.  The
        plan is unchanged -- same tensors, bytes and prefetch triggers -- only the D2H
        service order and, with it, the release of a deferred tensor move."""
        rw = self.rw
        g = rw.graph
        prod = {t: rw.position(g.tensor(t).producer) for t in swapped}
        if self.d2h_order == "fifo" or not swapped:
            order = sorted(swapped, key=lambda t: (prod[t], t))
            return {t: (prod[t], k) for k, t in enumerate(order)}
        need = {}
        for t in swapped:
            readers = [rw.position(c) for c in g.consumers(t + "@in") if c in rw._positions]
            need[t] = min(readers) if readers else len(rw.serial_order)
        starts, t0 = [], 0.0
        for nid in rw.serial_order:
            n = g.node(nid)
            rate = 8e14 if n.kind in ("conv", "upsample") else 9.6e13   # flop/s, 16 x B/s
            starts.append(t0)
            t0 += n.cost_units / rate
        ends = starts[1:] + [t0]
        ready = {t: ends[prod[t]] for t in swapped}
        link = 55e9
        left, order, tf = set(swapped), [], 0.0
        while left:
            avail = [t for t in left if ready[t] <= tf]
            if not avail:
                tf = min(ready[t] for t in left)
                continue
            t = min(avail, key=lambda u: (need[u], prod[u], u))
            order.append((t, tf))
            tf += nbytes[t] / link
            left.discard(t)
        out, last = {}, 0
        import bisect
        for k, (t, start) in enumerate(order):
            slot = max(prod[t], bisect.bisect_right(starts, start) - 1, last)
            # released (and so swapped out) no later than its prefetch trigger
            slot = min(slot, rw.position(swapped[t][2]))
            out[t] = (slot, k)
            last = max(last, slot)
        return out

    def _insert_grad_buckets(self):
        """Data parallel: mean of the per-rank gradients (NCCL over NVLink, BN statistics
        stay local), as ~dp_bucket_mb contiguous buckets of the flat gradient buffer.  A
        bucket's ALLREDUCE is placed right after the op that writes the last of its
        gradients, so it runs on the comm stream while the backward continues;
        the flat layout is in forward order, so walking it from the end follows the
        backward's completion order."""
        cfg, pr, lay = self.cfg, self.program, self.layout
        off2slot = {slot.offset: name for name, slot in lay.slots.items()}
        done = {}
        for k, (code, tids, ia, fa) in enumerate(pr.ops):
            if code in (OP["US_OP_CONV_WGRAD"], OP["US_OP_CONVT_WGRAD"]):
                done[off2slot[ia[6]]] = k
            elif code == OP["US_OP_BN_BWD"]:
                done[off2slot[ia[4]]] = k
                done[off2slot[ia[5]]] = k
            elif code == OP["US_OP_LOSS_BWD"]:
                done[off2slot[ia[6]]] = k
                done[off2slot[ia[7]]] = k
        opt_slot = len(self.rw.serial_order)
        adam = next(k for k, op in enumerate(pr.ops)
                    if op[0] == OP["US_OP_SLOT_BEGIN"] and op[2][0] == opt_slot)
        slots = sorted(lay.slots.items(), key=lambda kv: kv[1].offset)
        target = max(1, int(cfg.dp_bucket_mb * (1 << 20) / 4))
        buckets, end, cur = [], lay.total, []
        for name, slot in reversed(slots):
            cur.append(name)
            if end - slot.offset >= target or slot.offset == 0:
                ready = max(done.get(nm, adam - 1) for nm in cur)
                buckets.append((ready, slot.offset, end - slot.offset))
                end, cur = slot.offset, []
        self.grad_buckets = sorted(buckets)
        scale = 1.0 / max(1, cfg.world)
        reduce = cfg.world > 1 or cfg.dp_force_allreduce
        for ready, off, count in sorted(buckets, key=lambda b: (-b[0], -b[1])):
            # per bucket on the comm stream: [all-reduce], then the Adam update of exactly
            # these parameters -- their forward and backward uses are all behind them
            seq = []
            if reduce:
                seq.append((OP["US_OP_ALLREDUCE"], (self.t_G,), (off, count, 1), (scale,)))
            seq.append((OP["US_OP_ADAM"], (self.t_P, self.t_G, self.t_M, self.t_V, self.t_PB),
                        (count, 1 if cfg.dtype == "bf16" else 0, off, 1),
                        (cfg.lr, cfg.betas[0], cfg.betas[1], cfg.adam_eps, 1.0)))
            pr.ops[ready + 1:ready + 1] = seq

    # ------------------------------------------------------------------ data parallel
    def init_data_parallel(self, rank: int, world: int):
        """Create this rank's NCCL communicator from a unique id broadcast over
        torch.distributed (which must be initialised)."""
        import os
        if world <= 1 and not self.cfg.dp_force_allreduce:
            return
        if "US_NCCL_LIB" not in os.environ:
            try:
                import nvidia.nccl
                libdir = os.path.join(list(nvidia.nccl.__path__)[0], "lib")
                os.environ["US_NCCL_LIB"] = os.path.join(libdir, "libnccl.so.2")
            except Exception:
                pass
        if world <= 1:   # single-rank communicator (exercises the NCCL path on one GPU)
            self.engine.dp_init(Engine.nccl_unique_id(), 1, 0)
            return
        import torch.distributed as dist
        obj = [Engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        self.engine.dp_init(obj[0], world, rank)

    # ------------------------------------------------------------------ running
    def synthetic_batch(self, seed: int = 0):
        """BraTS-shaped synthetic input (N,4,D,H,W fp32, reference input recipe
        numeric.py:49-59) and uint8 labels in [0, n_classes)."""
        cfg = self.cfg
        D, H, W = cfg.dims
        rng = np.random.default_rng((seed, zlib.crc32(b"source")))
        x = rng.standard_normal(cfg.batch * cfg.in_channels * D * H * W).astype(np.float32)
        x = x.reshape(cfg.batch, cfg.in_channels, D, H, W)
        lrng = np.random.default_rng((seed, zlib.crc32(b"label")))
        y = lrng.integers(0, cfg.n_classes, size=(cfg.batch, D, H, W)).astype(np.uint8)
        return x, y

    def load_batch(self, x: np.ndarray, y: np.ndarray):
        self.engine.upload(self.t_IN, np.ascontiguousarray(x, np.float32))
        self.engine.upload(self.t_LBL, np.ascontiguousarray(y, np.uint8))

    def load_batch_ptr(self, x_ptr: int, y_ptr: int):
        """Upload from (pinned) host pointers: the e2e path of bench.py."""
        cfg = self.cfg
        vox = int(np.prod(cfg.dims)) * cfg.batch
        self.engine.upload_ptr(self.t_IN, x_ptr, vox * cfg.in_channels * 4)
        self.engine.upload_ptr(self.t_LBL, y_ptr, vox)

    def _set_adam_step(self):
        # Adam's bias correction depends on the step count: patch the op's fargs.
        self.step_count += 1
        for k in self._adam_engine_index:
            self.engine.set_farg(k, 4, float(self.step_count))

    def set_augmentation(self, flips: int, perm: int):
        """This step's augmentation: flip mask (bit 0 x, 1 y, 2 z) and axis permutation
        (index into (z,y,x) orders, csrc/elementwise.cu c_aug_perm)."""
        if not self.cfg.augment:
            raise GraphError("trainer built without augment=True")
        if perm not in self.aug_perms:
            raise GraphError(f"permutation {perm} does not preserve the volume shape")
        for k, (code, *_ ) in enumerate(self.program.ops):
            if code in (OP["US_OP_INPUT_NCDHW"], OP["US_OP_LABELS_AUG"]):
                self.engine.set_farg(k, 0, float(flips))
                self.engine.set_farg(k, 1, float(perm))
        self._aug_fixed = True

    def _draw_augmentation(self):
        if not self.cfg.augment or getattr(self, "_aug_fixed", False):
            return
        if not hasattr(self, "_aug_rng"):
            self._aug_rng = np.random.default_rng((self.cfg.seed, 0xA06))
        flips = int(self._aug_rng.integers(0, 8))
        perm = int(self.aug_perms[self._aug_rng.integers(0, len(self.aug_perms))])
        self.set_augmentation(flips, perm)
        self._aug_fixed = False

    @property
    def aug_perms(self) -> list:
        """Axis permutations (of z, y, x) that keep the volume's shape."""
        perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
        d = self.cfg.dims
        return [k for k, p in enumerate(perms) if all(d[p[i]] == d[i] for i in range(3))]

    def run_async(self):
        self._set_adam_step()
        self._draw_augmentation()
        try:
            self.engine.run()
        except EngineError as exc:
            _raise(exc)

    def step(self, x=None, y=None) -> dict:
        if x is not None:
            self.load_batch(x, y)
        self.run_async()
        try:
            self.engine.sync()
        except EngineError as exc:
            _raise(exc)
        st = self.engine.stats()
        loss = float(self.engine.download(self.t_LOSS, 4, np.float32)[0])
        return {"loss": loss, "step_s": st["step_s"], "stall_s": st["stall_s"],
                "d2h_bytes": st["d2h_bytes"], "h2d_bytes": st["h2d_bytes"],
                "arena_peak_bytes": st["arena_peak_bytes"], "kernels": st["kernels"]}

    # ------------------------------------------------------------------ results
    def params_now(self) -> dict:
        return self.unflat(self.engine.download(self.t_P, self.layout.total * 4, np.float32))

    def grads_now(self) -> dict:
        return self.unflat(self.engine.download(self.t_G, self.layout.total * 4, np.float32))

    def bn_stats(self) -> dict:
        """Saved BatchNorm batch statistics of the last step: norm id -> (mean, rstd)."""
        raw = self.engine.download(self.t_STAT, max(1, self.stat_total) * 4, np.float32)
        out = {}
        for nid, off in self.bn_off.items():
            c = self._chan(self.graph.node(nid).outputs[0])
            out[nid] = (raw[off:off + c].copy(), raw[off + c:off + 2 * c].copy())
        return out

    def dice_sums(self) -> np.ndarray:
        return self.engine.download(self.t_DICE, (3 * self.cfg.n_classes + 1) * 8, np.float64)

    def captured_tensor(self, t: str) -> np.ndarray:
        from .ops import from_bf16_bits
        tt = self.graph.tensor(t[2:] if t.startswith("d:") else t)
        shape = (self.cfg.batch,) + tuple(tt.shape) + (tt.channels,)
        nb = self.program.tensors["<capture>" + t].nbytes
        raw = self.engine.download(self.captured[t], nb, np.uint8)
        v = from_bf16_bits(raw.view(np.uint16)) if self.cfg.dtype == "bf16" else raw.view(np.float32)
        return v.reshape(shape)

    def timeline(self) -> SimReport:
        """The measured step as a reference-shaped SimReport (sim.py:76-96): compute
        slots, D2H/H2D copies and compute-stream stalls, in seconds.  A slot's compute
        event starts after the residency waits it opened with (the simulator's "compute
        starts when its inputs are resident"); the wait is the stall before it."""
        pr = self.program
        events, stalls = [], []
        busy = {"compute": 0.0, "d2h": 0.0, "h2d": 0.0}
        raw = self.engine.timeline()
        stall_end = {}
        for node, ch, s, e in raw:
            if ch == CH_STALL:
                stall_end[node] = max(stall_end.get(node, s), e)
        for node, ch, s, e in raw:
            if ch == CH_OP:
                continue
            if ch == CH_STALL:
                name = pr.slot_names.get(node, "optimizer")
                stalls.append((name, "copy", e - s))
                continue
            chan = {CH_COMPUTE: "compute", CH_D2H: "d2h", CH_H2D: "h2d"}[ch]
            if ch == CH_COMPUTE:
                name = pr.slot_names.get(node, "optimizer")
                s = min(max(s, stall_end.get(node, s)), e)
            else:
                name = pr.io_names.get(node, f"io{node}")
            events.append((name, chan, s, e))
            busy[chan] += e - s
        events.sort(key=lambda ev: (ev[2], {"compute": 0, "d2h": 1, "h2d": 2}[ev[1]], ev[0]))
        makespan = max((e for _, _, _, e in events), default=0.0)
        phases = {n.id: n.phase for n in self.rw.graph.nodes}
        phases["optimizer"] = "backward"
        st = self.engine.stats()
        return SimReport(makespan=makespan, events=events, peak_resident=st["arena_peak_bytes"],
                         stalls=stalls, busy={k: (v / makespan if makespan else 0.0)
                                              for k, v in busy.items()},
                         phases=phases)

    def physical_peak(self, rep: SimReport | None = None) -> int:
        """HBM the step tensors physically occupy at the worst moment of a measured step.

        The engine's arena peak counts a swapped tensor's block as free once the program
        releases it, but its bytes stay on the device until the D2H copy finishes (a
        block reused earlier makes the allocating stream wait).  From the timeline: a
        tensor lives from the start of the slot that first writes it (a prefetched copy:
        from its H2D start) to the end of the slot that frees it, or for a released
        tensor to the later of that and the end of its D2H copy."""
        rep = rep or self.timeline()
        pr = self.program
        inv = {v: k[len("US_OP_"):] for k, v in OP.items() if k.startswith("US_OP_")}
        start, end, copy_start, copy_end = {}, {}, {}, {}
        for name, ch, a, b in rep.events:
            if ch == "compute":
                start[name], end[name] = a, b
            else:
                copy_start[name], copy_end[name] = a, b
        defs = pr.by_tid()
        io_of = {}
        for code, tids, ia, _ in pr.ops:
            if inv.get(code) in ("SWAP_OUT", "SWAP_IN"):
                io_of[(inv[code], tids[-1] if inv[code] == "SWAP_IN" else tids[0])] = \
                    pr.io_names.get(ia[0])
        born, dead, cur = {}, {}, None
        for code, tids, ia, _ in pr.ops:
            op = inv.get(code)
            if op == "SLOT_BEGIN":
                cur = pr.slot_names.get(ia[0], "optimizer")
                continue
            if op == "SLOT_END":
                continue
            t_end = end.get(cur, 0.0)
            if op == "FREE":
                dead[tids[0]] = t_end
            elif op == "SWAP_RELEASE":
                d2h = copy_end.get(io_of.get(("SWAP_OUT", tids[0])), t_end)
                dead[tids[0]] = max(t_end, d2h)
            elif op == "SWAP_IN":
                born.setdefault(tids[1], copy_start.get(io_of.get(("SWAP_IN", tids[1])), t_end))
            else:
                for t in tids:
                    if t >= 0 and defs[t].storage == ARENA:
                        born.setdefault(t, start.get(cur, 0.0))
        ev = []
        for t, b in born.items():
            nb = (defs[t].nbytes + 1023) // 1024 * 1024
            ev.append((b, nb))
            ev.append((dead.get(t, rep.makespan), -nb))
        ev.sort(key=lambda e: (e[0], e[1]))
        live = peak = 0
        for _, d in ev:
            live += d
            peak = max(peak, live)
        return peak

    def op_times(self, steps: int = 3) -> list:
        """Kernel time of every compute op, measured with CUDA events on the compute
        stream (after its residency waits) over ``steps`` extra steps.  Returns
        [(op index, opcode name, slot name, mean seconds)]."""
        from ._native import FLAG_OP_TIMES, OP
        inv = {v: k[len("US_OP_"):] for k, v in OP.items() if k.startswith("US_OP_")}
        slot_of, cur = {}, None
        for k, (code, _, ia, _) in enumerate(self.program.ops):
            if inv.get(code) == "SLOT_BEGIN":
                cur = ia[0]
            slot_of[k] = cur
        base = self.engine.flags
        self.engine.set_flags(base | FLAG_OP_TIMES)
        acc: dict[int, float] = {}
        try:
            for _ in range(steps):
                self.run_async()
                self.engine.sync()
                for node, ch, s, e in self.engine.timeline():
                    if ch == CH_OP:
                        acc[node] = acc.get(node, 0.0) + (e - s)
        finally:
            self.engine.set_flags(base)
        out = []
        for k in sorted(acc):
            code = self.program.ops[k][0]
            out.append((k, inv.get(code, str(code)),
                        self.program.slot_names.get(slot_of.get(k), "optimizer"), acc[k] / steps))
        return out

    def close(self):
        self.engine.close()


def _raise(exc: EngineError):
    from .numeric import _raise_domain
    _raise_domain(exc)
