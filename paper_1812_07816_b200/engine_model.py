"""Timeline model of the engine executing one lowered program (tuner's predictor).

The reference predicts a plan with its discrete-event simulator (sim.py:114-277):
compute in serial order, one D2H and one H2D FIFO, a swap-in issued at its
trigger and allocated when it starts, memory freed when a swap-out completes.
That model prices the *plan*; the engine runs a *program* lowered from it, and
the two differ on the B200 in ways that decide whether a budget binds:

* what exists at all -- fused NORM_ACT leaves dead BatchNorm outputs unwritten
  (when elided), the upsample writes straight into its concat, ReLU gradients
  are fused into their producers, workspaces (BN / split-K partials) live in the
  arena;
* when a swap-out is issued -- need order (unet.py ``_d2h_issue_slots``), not
  production order;
* when memory comes back -- a released tensor's block is reusable only once its
  D2H copy has finished, so a budget below the program-order peak turns into
  compute-stream waits (the engine's allocator waits on the copy event).

``predict`` walks the lowered program op by op with measured slot times and
measured link bandwidths and returns the step time, the compute-stream stalls
(copy waits + memory waits), the physical peak and whether the budget is
feasible at all.  It prices exactly the bytes the engine moves.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

from ._native import ARENA, OP

_SLOT_BEGIN, _SLOT_END = OP["US_OP_SLOT_BEGIN"], OP["US_OP_SLOT_END"]
_SWAP_OUT, _SWAP_IN = OP["US_OP_SWAP_OUT"], OP["US_OP_SWAP_IN"]
_RELEASE, _FREE = OP["US_OP_SWAP_RELEASE"], OP["US_OP_FREE"]
_NO_READ = {_SLOT_BEGIN, _SLOT_END, _SWAP_OUT, _SWAP_IN, _RELEASE, _FREE}


@dataclass
class Prediction:
    step_s: float
    compute_s: float
    stall_s: float                  # compute-stream waits (prefetch + memory pressure)
    copy_stall_s: float             # ... of which waiting for a prefetch
    memory_stall_s: float           # ... of which waiting for a swap-out to free memory
    physical_peak: int              # bytes resident at the worst moment (released-but-
                                    # not-yet-copied swap-outs included)
    d2h_bytes: int
    h2d_bytes: int
    feasible: bool
    reason: str = ""
    slot_start: dict = field(default_factory=dict)
    op_clock: list = field(default_factory=list)    # compute clock when op k is issued
    d2h_done: dict = field(default_factory=dict)    # tid -> end of its swap-out copy
    layout_peak: int = 0                            # max offset + size (static layout)

    @property
    def exposed(self) -> float:
        return self.stall_s / self.step_s if self.step_s > 0 else 0.0


def _rnd(n: int) -> int:
    return (n + 1023) // 1024 * 1024


def predict(program, slot_seconds: dict, d2h_bw: float, h2d_bw: float,
            budget: int | None = None, offsets: dict | None = None) -> Prediction:
    """Simulate one step of ``program`` (lowering.Program).

    slot_seconds: compute seconds per slot NAME (serial-order node id, "optimizer");
    slots missing from it cost 0.  budget: arena bytes (None = unlimited).  offsets:
    the static arena layout (Program.place) -- then an allocation waits exactly for the
    tensors released earlier in its region (a swap-out's region: until its D2H copy
    ends) and the budget check is the layout's extent; without it, memory is a byte
    count (the best-fit allocator, fragmentation ignored)."""
    if offsets is not None:
        return _predict_placed(program, slot_seconds, d2h_bw, h2d_bw, budget, offsets)
    defs = program.by_tid()
    budget = budget if budget else 1 << 62
    t = 0.0                       # compute-stream clock
    d2h_free = h2d_free = 0.0     # copy-engine clocks (one FIFO per direction)
    d2h_done: dict[int, float] = {}
    h2d_done: dict[int, float] = {}
    live: dict[int, int] = {}     # tid -> bytes held (allocated, not freed)
    pending: list = []            # heap of (d2h end, bytes) of released swap-outs
    in_use = 0                    # live + pending bytes
    peak = 0
    stall_copy = stall_mem = compute = 0.0
    d2h_bytes = h2d_bytes = 0
    cur = None
    slot_t0 = 0.0
    starts = {}
    waited_slot = set()

    def reclaim(now):
        nonlocal in_use
        while pending and pending[0][0] <= now:
            in_use -= heapq.heappop(pending)[1]

    def allocate(tid, now):
        """Bytes for tid at time `now`; returns the time the allocation can proceed."""
        nonlocal in_use, peak
        nb = _rnd(defs[tid].nbytes)
        reclaim(now)
        while in_use + nb > budget and pending:
            now = max(now, pending[0][0])
            reclaim(now)
        if in_use + nb > budget:
            return None
        in_use += nb
        live[tid] = nb
        peak = max(peak, in_use)
        return now

    op_clock = []
    for code, tids, ia, _ in program.ops:
        op_clock.append(t)
        if code == _SLOT_BEGIN:
            cur = program.slot_names.get(ia[0], "optimizer")
            slot_t0 = t
            starts[cur] = t
            continue
        if code == _SLOT_END:
            dt = float(slot_seconds.get(cur, 0.0))
            t += dt
            compute += dt
            continue
        if code == _SWAP_OUT:
            tid = tids[0]
            s = max(t, d2h_free)
            d2h_free = s + defs[tid].nbytes / d2h_bw
            d2h_done[tid] = d2h_free
            d2h_bytes += defs[tid].nbytes
            continue
        if code == _RELEASE:
            tid = tids[0]
            nb = live.pop(tid, 0)
            # the block stays resident until its D2H copy has finished
            heapq.heappush(pending, (d2h_done.get(tid, t), nb))
            continue
        if code == _FREE:
            in_use -= live.pop(tids[0], 0)
            continue
        if code == _SWAP_IN:
            src, dst = tids
            ready = max(t, h2d_free, d2h_done.get(src, t))
            got = allocate(dst, ready)
            if got is None:
                return Prediction(t, compute, stall_copy + stall_mem, stall_copy, stall_mem,
                                  peak, d2h_bytes, h2d_bytes, False,
                                  f"prefetch of {defs[dst].name} cannot fit the budget")
            h2d_free = got + defs[dst].nbytes / h2d_bw
            h2d_done[dst] = h2d_free
            h2d_bytes += defs[dst].nbytes
            continue
        if code in _NO_READ:
            continue
        # a compute op: wait for prefetched operands, allocate first-written tensors
        for tid in tids:
            if tid < 0:
                continue
            if tid in h2d_done and h2d_done[tid] > t:
                stall_copy += h2d_done[tid] - t
                t = h2d_done[tid]
                waited_slot.add(cur)
            if defs[tid].storage == ARENA and tid not in live and tid not in h2d_done:
                got = allocate(tid, t)
                if got is None:
                    return Prediction(t, compute, stall_copy + stall_mem, stall_copy,
                                      stall_mem, peak, d2h_bytes, h2d_bytes, False,
                                      f"{defs[tid].name} cannot fit the budget")
                if got > t:
                    stall_mem += got - t
                    t = got
    end = max(t, d2h_free, h2d_free)
    return Prediction(end, compute, stall_copy + stall_mem, stall_copy, stall_mem, peak,
                      d2h_bytes, h2d_bytes, True, slot_start=starts, op_clock=op_clock,
                      d2h_done=d2h_done)


def _predict_placed(program, slot_seconds, d2h_bw, h2d_bw, budget, offsets) -> Prediction:
    defs = program.by_tid()
    size = {t: _rnd(defs[t].nbytes) for t in offsets}
    extent = max((offsets[t] + size[t] for t in offsets), default=0)
    if budget and extent > budget:
        return Prediction(0.0, 0.0, 0.0, 0.0, 0.0, extent, 0, 0, False,
                          f"layout needs {extent} bytes > budget {budget}",
                          layout_peak=extent)
    t = 0.0
    d2h_free = h2d_free = 0.0
    d2h_done: dict[int, float] = {}
    h2d_done: dict[int, float] = {}
    freed = []          # (offset, end, time the region is reusable)
    live: dict[int, int] = {}
    in_use = peak = 0
    stall_copy = stall_mem = compute = 0.0
    d2h_bytes = h2d_bytes = 0
    cur = None
    starts, op_clock = {}, []

    def region_ready(tid):
        o, e = offsets[tid], offsets[tid] + size[tid]
        return max((r for a, b, r in freed if a < e and o < b), default=0.0)

    def take(tid):
        nonlocal in_use, peak
        live[tid] = size[tid]
        in_use += size[tid]
        peak = max(peak, in_use)

    for code, tids, ia, _ in program.ops:
        op_clock.append(t)
        if code == _SLOT_BEGIN:
            cur = program.slot_names.get(ia[0], "optimizer")
            starts[cur] = t
        elif code == _SLOT_END:
            dt = float(slot_seconds.get(cur, 0.0))
            t += dt
            compute += dt
        elif code == _SWAP_OUT:
            tid = tids[0]
            s0 = max(t, d2h_free)
            d2h_free = s0 + defs[tid].nbytes / d2h_bw
            d2h_done[tid] = d2h_free
            d2h_bytes += defs[tid].nbytes
        elif code in (_RELEASE, _FREE):
            tid = tids[0]
            if tid in live:
                in_use -= live.pop(tid)
                ready = d2h_done.get(tid, t) if code == _RELEASE else t
                freed.append((offsets[tid], offsets[tid] + size[tid], max(ready, t)))
        elif code == _SWAP_IN:
            src, dst = tids
            s0 = max(t, h2d_free, d2h_done.get(src, t), region_ready(dst))
            take(dst)
            h2d_free = s0 + defs[dst].nbytes / h2d_bw
            h2d_done[dst] = h2d_free
            h2d_bytes += defs[dst].nbytes
        elif code not in _NO_READ:
            for tid in tids:
                if tid < 0:
                    continue
                if tid in h2d_done and h2d_done[tid] > t:
                    stall_copy += h2d_done[tid] - t
                    t = h2d_done[tid]
                if tid in offsets and tid not in live and tid not in h2d_done:
                    r = region_ready(tid)
                    if r > t:
                        stall_mem += r - t
                        t = r
                    take(tid)
    end = max(t, d2h_free, h2d_free)
    return Prediction(end, compute, stall_copy + stall_mem, stall_copy, stall_mem, peak,
                      d2h_bytes, h2d_bytes, True, slot_start=starts, op_clock=op_clock,
                      d2h_done=d2h_done, layout_peak=extent)


def plan_layout(program, slot_seconds: dict, d2h_bw: float, h2d_bw: float,
                budget: int | None = None, slack: float = 1.25):
    """Static arena layout for ``program``, time-aware: a swapped-out tensor's region is
    held (not handed to a later tensor) until its D2H copy is predicted to be done, with
    ``slack`` on that time, so an unconstrained step never waits on a copy for memory.
    Under a budget the hold is shortened (1, 3/4, 1/2, 1/4, 0 of it) until the layout
    fits; what remains shows up as memory waits in ``predict``.  Returns (offsets, layout
    peak, hold fraction) or (None, peak, None) when even the program-order layout does
    not fit."""
    import bisect
    free = predict(program, slot_seconds, d2h_bw, h2d_bw)
    clock = free.op_clock
    release_at = {tids[0]: k for k, (code, tids, _, _) in enumerate(program.ops)
                  if code == _RELEASE}
    full = {}
    for tid, k in release_at.items():
        done = free.d2h_done.get(tid)
        if done is None:
            continue
        j = bisect.bisect_left(clock, done * slack)
        full[tid] = max(k, j)
    peak = None
    for frac in (1.0, 0.75, 0.5, 0.25, 0.0):
        hold = {t: release_at[t] + int(frac * (full[t] - release_at[t])) for t in full}
        offs, peak = program.place(program.lifetimes(hold))
        if not budget or peak <= budget:
            return offs, peak, frac
    return None, peak, None


# B200 rates of the reference cost units (models.py:14-39) for a first estimate when no
# measured slot times are at hand, fitted to the round-1 192^3 no-swap step: conv / convT
# (forward and gradient) 1.1e15 units/s, memory-bound ops 4.6e14 units/s (16 x B/s).
CONV_RATE, MEM_RATE = 1.1e15, 4.6e14


def estimate_slot_seconds(rw, clone_map=None) -> dict:
    """Compute seconds per serial slot of a (rewritten) training graph from the cost
    model at B200 rates; a recompute clone costs its original op."""
    g = rw.graph
    clone_map = clone_map or {}
    out = {}
    for nid in rw.serial_order:
        n = g.node(nid)
        base = g.node(clone_map[nid]) if nid in clone_map and g.has_node(clone_map[nid]) else n
        kind = base.kind
        if kind == "grad":
            kind = g.node(rw.grad_of[nid]).kind
        out[nid] = base.cost_units / (CONV_RATE if kind in ("conv", "upsample") else MEM_RATE)
    return out


def slot_times_from_timeline(rep, scale: float = 1.0) -> dict:
    """Measured compute seconds per slot name from a SimReport-shaped timeline
    (UNetTrainer.timeline())."""
    out: dict[str, float] = {}
    for name, ch, s, e in rep.events:
        if ch == "compute":
            out[name] = out.get(name, 0.0) + scale * (e - s)
    return out
