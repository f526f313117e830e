"""Compile a TrainingGraph + RewritePlan into a libunetswap program.

A program is a flat list of device ops (see csrc/opcodes.h) over integer
tensor ids.  This module owns the *placement* rules that make the GPU step
execute the reference planner's schedule:

* compute slots follow ``tg.serial_order`` (training.py:139), one
  SLOT_BEGIN/SLOT_END pair per serial position;
* a swapped tensor's D2H copy is issued right after its producer (the
  simulator's "ready when the producer completes", sim.py:229-236) and its
  device memory is released at the reference's swap_out anchor -- after the
  last forward reader (numeric.py:122-129);
* its H2D prefetch is issued right after the trigger slot ends
  (numeric.py:130-136, rewrite.py:177), in (trigger, earliest reader, id)
  order, which is the simulator's H2D FIFO key (sim.py:289-293);
* every other step tensor is freed after its last reader.

``lower_toy`` reproduces the reference's toy executor (numeric.py:153-276)
op for op; the real U-Net lowering lives in ``unet.py`` and uses the same
``Program`` container and placement helpers.
"""
from __future__ import annotations

import zlib
from dataclasses import dataclass, field

import numpy as np

from ._native import ARENA, DT_F64, OP, PERSIST
from .graph import GraphError, element_count
from .training import TrainingGraph

AFFINE_KINDS = ("conv", "matmul", "upsample", "source", "sink", "recompute")

# ops whose operands are not ordinary reads/writes for liveness purposes
_IO_OPS = {OP["US_OP_SLOT_BEGIN"], OP["US_OP_SLOT_END"], OP["US_OP_SWAP_RELEASE"],
           OP["US_OP_FREE"]}


@dataclass
class TensorDef:
    tid: int
    name: str
    nbytes: int
    storage: int
    dtype: int


@dataclass
class Program:
    """Host-side record of a libunetswap program (emitted with ``emit``)."""

    tensors: dict = field(default_factory=dict)      # name -> TensorDef
    ops: list = field(default_factory=list)          # (opcode, tids, iargs, fargs)
    slot_names: dict = field(default_factory=dict)   # slot id -> node id
    io_names: dict = field(default_factory=dict)     # io id -> io node id
    slot_phase: dict = field(default_factory=dict)   # slot id -> phase

    def tensor(self, name: str, nbytes: int, storage: int = ARENA, dtype: int = DT_F64) -> int:
        if name in self.tensors:
            raise GraphError(f"program tensor {name!r} defined twice")
        tid = len(self.tensors)
        self.tensors[name] = TensorDef(tid, name, int(nbytes), storage, dtype)
        return tid

    def tid(self, name: str) -> int:
        return self.tensors[name].tid

    def op(self, opname: str, tids=(), iargs=(), fargs=()):
        self.ops.append((OP["US_OP_" + opname], tuple(int(t) for t in tids),
                         tuple(int(v) for v in iargs), tuple(float(v) for v in fargs)))

    def by_tid(self) -> dict:
        return {d.tid: d for d in self.tensors.values()}

    def insert_frees(self, keep=()):
        """Append FREE after the last use of every step tensor not released by a swap."""
        defs = self.by_tid()
        released = {tids[0] for code, tids, _, _ in self.ops if code == OP["US_OP_SWAP_RELEASE"]}
        keep_ids = {self.tid(n) for n in keep}
        last: dict[int, int] = {}
        for k, (code, tids, _, _) in enumerate(self.ops):
            if code in _IO_OPS:
                continue
            for t in tids:
                if t >= 0 and defs[t].storage == ARENA:
                    last[t] = k
        frees: dict[int, list[int]] = {}
        for t, k in last.items():
            if t in released or t in keep_ids:
                continue
            frees.setdefault(k, []).append(t)
        out = []
        for k, entry in enumerate(self.ops):
            out.append(entry)
            for t in sorted(frees.get(k, ())):
                out.append((OP["US_OP_FREE"], (t,), (), ()))
        self.ops = out

    def emit(self, engine, offsets=None):
        engine.reset()
        for d in sorted(self.tensors.values(), key=lambda d: d.tid):
            engine.tensor(d.tid, d.nbytes, d.storage, d.dtype, d.name)
        for tid, off in sorted((offsets or {}).items()):
            engine.place(tid, off)
        for slot, name in self.slot_names.items():
            engine.slot_name(slot, name)
        for code, tids, iargs, fargs in self.ops:
            engine.op(code, tids, iargs, fargs)
        engine.finalize()

    def order_peak(self) -> int:
        """Peak of live step-tensor bytes in program order (the engine's arena peak
        before fragmentation): allocated at first write or prefetch, returned at FREE or
        SWAP_RELEASE."""
        defs = self.by_tid()
        live, cur, peak = set(), 0, 0
        rnd = lambda t: (defs[t].nbytes + 1023) // 1024 * 1024
        for code, tids, _, _ in self.ops:
            if code in (OP["US_OP_FREE"], OP["US_OP_SWAP_RELEASE"]):
                if tids[0] in live:
                    live.discard(tids[0])
                    cur -= rnd(tids[0])
                continue
            if code in (OP["US_OP_SLOT_BEGIN"], OP["US_OP_SLOT_END"], OP["US_OP_SWAP_OUT"]):
                continue
            targets = tids[1:2] if code == OP["US_OP_SWAP_IN"] else tids
            for t in targets:
                if t >= 0 and defs[t].storage == ARENA and t not in live:
                    live.add(t)
                    cur += rnd(t)
                    peak = max(peak, cur)
        return peak

    def lifetimes(self, hold_until=None) -> dict:
        """tid -> (first op index, last op index) of every arena tensor in program order:
        from its first write (a prefetch: its SWAP_IN) to its FREE / SWAP_RELEASE.  A
        released (swapped-out) tensor may be held longer -- ``hold_until[tid]`` -- so its
        region is not handed out while its D2H copy is still reading it."""
        defs = self.by_tid()
        hold_until = hold_until or {}
        start, end = {}, {}
        skip = (OP["US_OP_SLOT_BEGIN"], OP["US_OP_SLOT_END"], OP["US_OP_SWAP_OUT"])
        for k, (code, tids, _, _) in enumerate(self.ops):
            if code in skip:
                continue
            if code == OP["US_OP_FREE"]:
                end[tids[0]] = k
            elif code == OP["US_OP_SWAP_RELEASE"]:
                end[tids[0]] = max(k, hold_until.get(tids[0], k))
            elif code == OP["US_OP_SWAP_IN"]:
                start.setdefault(tids[1], k)
            else:
                for t in tids:
                    if t >= 0 and defs[t].storage == ARENA:
                        start.setdefault(t, k)
        n = len(self.ops)
        return {t: (a, end.get(t, n)) for t, a in start.items()}

    def place(self, lifetimes: dict) -> tuple[dict, int]:
        """Static arena layout: offsets such that tensors whose lifetimes overlap never
        share bytes.  Greedy by size (largest first, lowest free offset among the
        conflicting tensors already placed), 1 KiB granularity.  Returns (tid -> offset,
        layout peak bytes)."""
        defs = self.by_tid()
        rnd = lambda t: max(1024, (defs[t].nbytes + 1023) // 1024 * 1024)   # noqa: E731
        order = sorted(lifetimes, key=lambda t: (-rnd(t), lifetimes[t][0], t))
        placed = []   # (offset, size, start, end)
        offs, peak = {}, 0
        for t in order:
            a, b = lifetimes[t]
            size = rnd(t)
            busy = sorted((o, o + sz) for o, sz, s0, e0 in placed if s0 <= b and a <= e0)
            off = 0
            for o, e in busy:
                if o - off >= size:
                    break
                off = max(off, e)
            offs[t] = off
            placed.append((off, size, a, b))
            peak = max(peak, off + size)
        return offs, peak

    def arena_need(self) -> int:
        return sum((d.nbytes + 1023) // 1024 * 1024 for d in self.tensors.values()
                   if d.storage == ARENA)


# ---------------------------------------------------------------------------
# Placement shared by the toy and the real lowering

@dataclass
class SwapSchedule:
    """Where the plan's io nodes go around the serial compute slots."""

    release_after: dict   # serial position -> [tensor id] (device copy released)
    prefetch_after: dict  # serial position -> [(tensor id, io node id)] in H2D FIFO order
    swapped: dict         # tensor id -> (swap_out id, swap_in id, trigger)


def swap_schedule(tg: TrainingGraph, plan) -> SwapSchedule:
    g = tg.graph
    pos = tg._positions
    release: dict[int, list[str]] = {}
    prefetch: dict[int, list[tuple]] = {}
    swapped = dict(plan.swapped) if plan is not None else {}
    for n in g.nodes:
        if n.kind == "swap_out":
            tid = n.inputs[0]
            anchor = pos[g.tensor(tid).producer]
            for c in g.consumers(tid):
                if g.has_node(c) and g.node(c).phase == "forward" and c in pos:
                    anchor = max(anchor, pos[c])
            release.setdefault(anchor, []).append(tid)
        elif n.kind == "swap_in":
            triggers = [a for a, b in g.control_edges
                        if b == n.id and g.node(a).kind != "swap_out"]
            if not triggers:
                raise GraphError(f"swap_in {n.id!r} has no trigger control edge")
            anchor = max(pos[t] for t in triggers)
            src = n.outputs[0][:-len("@in")]
            readers = [pos[c] for c in g.consumers(n.outputs[0]) if c in pos]
            prefetch.setdefault(anchor, []).append((min(readers) if readers else 0, n.id, src))
    for k in release:
        release[k].sort()
    pre = {k: [(src, nid) for _, nid, src in sorted(v)] for k, v in prefetch.items()}
    return SwapSchedule(release_after=release, prefetch_after=pre, swapped=swapped)


# ---------------------------------------------------------------------------
# Toy lowering: the reference executor's arithmetic on the GPU in fp64

def node_params(node_id: str) -> tuple[float, float]:
    """Per-op affine coefficients of the reference toy executor (numeric.py:36-41)."""
    h = zlib.crc32(node_id.encode())
    return 0.7 + 0.6 * ((h & 0xFFFF) / 0xFFFF), -0.5 + ((h >> 16) / 0xFFFF)


def input_values(g, seed: int, overrides=None) -> dict:
    """Seeded N(0,1) inputs per source node (reference numeric.py:49-59)."""
    vals = {}
    for n in g.nodes:
        if n.phase == "forward" and not n.inputs and n.outputs:
            tid = n.outputs[0]
            if overrides and tid in overrides:
                vals[tid] = np.asarray(overrides[tid], dtype=np.float64).copy()
            else:
                rng = np.random.default_rng((seed, zlib.crc32(n.id.encode())))
                vals[tid] = rng.standard_normal(element_count(g.tensor(tid)))
    return vals


@dataclass
class ToyLowering:
    program: Program
    inputs: dict        # graph input tensor -> (staging tid, values)
    results: dict       # graph input tensor -> result tid
    loss_tid: int
    act_inputs: dict = field(default_factory=dict)   # activation input -> captured tid


def lower_toy(tg: TrainingGraph, plan=None, seed: int = 0, inputs=None,
              capture_activation_inputs: bool = False) -> ToyLowering:
    """capture_activation_inputs: also copy out every forward activation's input (the
    kink distance grad_check resamples on, reference numeric.py:325-358)."""
    g = tg.graph
    pr = Program()
    n_el = {t.id: element_count(t) for t in g.tensors}
    for t in g.tensors:
        pr.tensor(t.id, n_el[t.id] * 8)
    loss_t = pr.tensor("<loss>", 8, PERSIST)
    vals = input_values(g, seed, inputs)
    staged = {tid: (pr.tensor("<input>" + tid, v.nbytes, PERSIST), v) for tid, v in vals.items()}
    results = {}
    for n in g.nodes:
        if n.phase == "forward" and not n.inputs and n.outputs:
            gid = f"grad/{n.id}:0"
            if g.has_tensor(gid):
                results[n.outputs[0]] = pr.tensor("<result>" + n.outputs[0], n_el[gid] * 8, PERSIST)
    loss_node = next((n for n in g.nodes if n.kind == "loss"), None)
    loss_inputs = set(loss_node.inputs) if loss_node else set()
    sched = swap_schedule(tg, plan)
    io_ids = {}
    act_inputs = {}

    def T(name):
        return pr.tid(name)

    def scratch(name, count):
        return pr.tensor(name, count * 8)

    for p, nid in enumerate(tg.serial_order):
        n = g.node(nid)
        pr.slot_names[p] = nid
        pr.slot_phase[p] = n.phase
        pr.op("SLOT_BEGIN", (), (p, 0 if n.phase == "forward" else 1))
        if n.kind == "loss":
            for k, tid in enumerate(n.inputs):
                pr.op("TOY_SUMSQ", (T(tid), loss_t), (n_el[tid], 1 if k == 0 else 0, 0))
        elif n.kind == "grad":
            _toy_grad(pr, tg, n, n_el, loss_inputs, scratch)
        elif not n.inputs:
            if n.outputs and n.outputs[0] in staged:
                out = n.outputs[0]
                pr.op("COPY_IN", (staged[out][0], T(out)), (n_el[out] * 8,))
        else:
            _toy_forward(pr, g, n, n_el)
            if capture_activation_inputs and n.kind == "activation" and n.phase == "forward":
                x = n.inputs[0]
                if x not in act_inputs:
                    act_inputs[x] = pr.tensor("<kink>" + x, n_el[x] * 8, PERSIST)
                    pr.op("CAPTURE", (T(x), act_inputs[x]), (n_el[x] * 8, 0))
        # D2H of swapped outputs leaves as soon as the producer is done
        for out in n.outputs:
            if out in sched.swapped:
                io = len(io_ids)
                io_ids[sched.swapped[out][0]] = io
                pr.io_names[io] = sched.swapped[out][0]
                pr.op("SWAP_OUT", (T(out),), (io,))
        pr.op("SLOT_END", (), (p,))
        for tid in sched.release_after.get(p, ()):
            pr.op("SWAP_RELEASE", (T(tid),))
        for src, in_node in sched.prefetch_after.get(p, ()):
            io = len(io_ids)
            io_ids[in_node] = io
            pr.io_names[io] = in_node
            pr.op("SWAP_IN", (T(src), T(src + "@in")), (io, p))
        if n.kind == "grad":
            for src_t, res in results.items():
                gid = f"grad/{g.tensor(src_t).producer}:0"
                if gid in n.outputs:
                    pr.op("CAPTURE", (T(gid), res), (n_el[gid] * 8, 0))
    pr.insert_frees()
    return ToyLowering(program=pr, inputs={k: v for k, v in staged.items()},
                       results=results, loss_tid=loss_t, act_inputs=act_inputs)


def _toy_forward(pr: Program, g, n, n_el):
    xs = list(n.inputs)
    out = n.outputs[0]
    T = pr.tid
    base = n.id.split("@rc")[0]
    if n.kind in AFFINE_KINDS:
        a, b = node_params(base)
        pr.op("TOY_AFFINE", (T(xs[0]), T(out)), (n_el[xs[0]], n_el[out]), (a, b))
    elif n.kind == "activation":
        pr.op("TOY_RELU", (T(xs[0]), T(out)), (n_el[out],))
    elif n.kind == "norm":
        pr.op("TOY_CENTER", (T(xs[0]), T(out)), (n_el[out],))
    elif n.kind == "pool":
        k = n_el[xs[0]] // n_el[out]
        if k * n_el[out] != n_el[xs[0]]:
            raise GraphError(f"pool {n.id!r}: input size not a multiple of the output size")
        pr.op("TOY_POOL", (T(xs[0]), T(out)), (n_el[out], k))
    elif n.kind == "concat":
        off = 0
        for x in xs:
            pr.op("TOY_COPY", (T(x), T(out)), (n_el[x], 0, off))
            off += n_el[x]
    else:
        raise GraphError(f"no toy semantic for node kind {n.kind!r}")


def _toy_grad(pr: Program, tg: TrainingGraph, n, n_el, loss_inputs, scratch):
    g = tg.graph
    T = pr.tid
    f = g.node(tg.grad_of[n.id])
    contribs, reuse = [], None
    for tid in n.inputs:
        if g.node(g.tensor(tid).producer).kind == "grad":
            contribs.append(tid)
        else:
            reuse = tid
    if reuse is None:
        raise GraphError(f"grad node {n.id!r} lacks its reuse-edge input")
    pr.op("TOUCH", (T(reuse),))   # the reference reads the reuse tensor in every grad slot
    size = n_el[reuse]
    fed_loss = bool(f.outputs) and f.outputs[0] in loss_inputs
    if not contribs or len(contribs) > 1 or fed_loss:
        inc = scratch(f"<incoming>{n.id}", size)
        if not contribs:
            pr.op("ZERO", (inc,))
        elif len(contribs) == 1:
            pr.op("TOY_COPY", (T(contribs[0]), inc), (size, 0, 0))
        else:
            pr.op("TOY_ADD", (T(contribs[0]), T(contribs[1]), inc), (size,), (1.0,))
            for c in contribs[2:]:
                pr.op("TOY_ADD", (inc, T(c), inc), (size,), (1.0,))
        if fed_loss:
            pr.op("TOY_ADD", (inc, T(reuse), inc), (size,), (2.0,))
    else:
        inc = T(contribs[0])
    outs = list(n.outputs)
    kind = f.kind
    if not f.inputs:
        pr.op("TOY_COPY", (inc, T(outs[0])), (size, 0, 0))
    elif kind in AFFINE_KINDS:
        a, _ = node_params(f.id)
        pr.op("TOY_AFFINE_BWD", (inc, T(outs[0])), (n_el[outs[0]], size), (a,))
    elif kind == "activation":
        pr.op("TOY_RELU_BWD", (inc, T(reuse), T(outs[0])), (size,))
    elif kind == "norm":
        pr.op("TOY_CENTER", (inc, T(outs[0])), (size,))
    elif kind == "pool":
        k = n_el[outs[0]] // size
        pr.op("TOY_POOL_BWD", (inc, T(outs[0])), (n_el[outs[0]], k))
    elif kind == "concat":
        off = 0
        for o in outs:
            pr.op("TOY_COPY", (inc, T(o)), (n_el[o], off, 0))
            off += n_el[o]
    else:
        raise GraphError(f"no toy gradient for node kind {kind!r}")
