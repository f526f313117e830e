"""Timeline model and report shape for swapped training steps.

Drop-in for ``pkg/src/swapsim/sim.py``.  ``simulate`` (sim.py:114-305) is
the discrete-event model of the channels the CUDA engine really has: one
compute stream running the serial order, a FIFO D2H copy stream (served by
ready time, then producer position) and a FIFO H2D copy stream (served in
trigger-issue order, head-of-line waiting on its own D2H).  The engine's
measured timeline is returned in the same ``SimReport`` shape
(``paper_1812_07816_b200.unet.UNetTrainer.timeline``), so ``stall_report``
(sim.py:308-325) gives the *measured* exposed-swap split as well as the
modelled one, and ``emit_trace`` writes either as a Chrome trace.
"""
from __future__ import annotations

import heapq
import json
from dataclasses import dataclass

from .graph import GraphError, NodeSpec, tensor_bytes
from .training import TrainingGraph

CHANNELS = ("compute", "d2h", "h2d")
_PRIO = {"compute": 0, "d2h": 1, "h2d": 2}
TRACE_TIDS = {"compute": 0, "d2h": 1, "h2d": 2}


class InfeasibleError(GraphError):
    def __init__(self, tensor_id: str, nbytes: int, budget: int):
        super().__init__(f"infeasible: tensor {tensor_id!r} needs {nbytes} bytes, "
                         f"which can never fit in the {budget}-byte budget")
        self.tensor_id = tensor_id


class DeadlockError(GraphError):
    def __init__(self, waiting: list, detail: str):
        super().__init__(f"simulation deadlock; waiting nodes: {waiting}; {detail}")
        self.waiting = waiting


@dataclass
class SimConfig:
    compute_rate: float = 1e12
    d2h_bw: float = 40e9
    h2d_bw: float = 40e9
    xfer_latency: float = 0.0
    gpu_budget: int = 0
    static_bytes: int = 0
    enforce_budget: bool = False

    def validate(self) -> None:
        if min(self.compute_rate, self.d2h_bw, self.h2d_bw) <= 0:
            raise GraphError("compute_rate and bandwidths must be positive")
        if self.xfer_latency < 0:
            raise GraphError("xfer_latency must be >= 0")


def op_cost(n: NodeSpec, cfg: SimConfig) -> float:
    return 0.0 if n.kind in ("swap_out", "swap_in") else n.cost_units / cfg.compute_rate


def xfer_cost(nbytes: int, bw: float, latency: float = 0.0) -> float:
    if bw <= 0:
        raise GraphError("bandwidth must be positive")
    return latency + nbytes / bw


@dataclass
class SimReport:
    makespan: float
    events: list        # (node id, channel, start, end)
    peak_resident: int
    stalls: list        # (waiting node, blocking node or "budget", duration)
    busy: dict
    phases: dict

    def to_obj(self) -> dict:
        return {"version": 1, "makespan": self.makespan, "peak_resident": self.peak_resident,
                "events": [list(e) for e in self.events],
                "stalls": [list(s) for s in self.stalls],
                "busy": dict(sorted(self.busy.items()))}

    def to_json(self) -> str:
        return json.dumps(self.to_obj(), sort_keys=True, indent=2) + "\n"


def peak_from_deltas(deltas) -> int:
    """Peak of a resident-bytes trace; same-instant deltas are netted first."""
    net: dict[float, int] = {}
    for when, d in deltas:
        net[when] = net.get(when, 0) + d
    peak = cur = 0
    for when in sorted(net):
        cur += net[when]
        if cur > peak:
            peak = cur
    return peak


class _Timeline:
    """Event-driven executor of one training step over three channels."""

    def __init__(self, tg: TrainingGraph, cfg: SimConfig):
        self.tg, self.cfg, self.g = tg, cfg, tg.graph
        g = self.g
        self.waits = {n.id: 0 for n in g.nodes}        # unfinished predecessors
        self.succ: dict[str, list[str]] = {n.id: [] for n in g.nodes}
        self.trigger_waits = {n.id: 0 for n in g.nodes if n.kind == "swap_in"}
        for a, b in g.edges():
            self.waits[b] += 1
            self.succ[a].append(b)
            if b in self.trigger_waits and g.node(a).kind != "swap_out":
                self.trigger_waits[b] += 1
        self.readers_left = {t.id: len(g.consumers(t.id)) for t in g.tensors}
        self.size = {t.id: tensor_bytes(t) for t in g.tensors}
        self.serial = list(tg.serial_order)
        pos = tg._positions
        self.queue_pos: dict[str, int] = {}
        for n in g.nodes:
            if n.kind == "swap_in":
                readers = [pos[c] for t in n.outputs for c in g.consumers(t) if c in pos]
                self.queue_pos[n.id] = min(readers) if readers else 0
            elif n.kind == "swap_out":
                prod = g.tensor(n.inputs[0]).producer
                self.queue_pos[n.id] = pos[prod] if prod in pos else 0
        self.last_dep: dict[str, tuple[float, str]] = {}
        self.resident = 0
        self.deltas: list[tuple[float, int]] = []
        self.events: list = []
        self.stalls: list = []
        self.inflight: list = []
        self.d2h_q: list = []
        self.h2d_q: list = []
        self.idle = {c: True for c in CHANNELS}
        self.busy_t = {c: 0.0 for c in CHANNELS}
        self.next_compute = 0
        self.compute_free_at = 0.0
        self.budget_blocked = False

    # memory ---------------------------------------------------------------
    def _fits(self, extra: int) -> bool:
        c = self.cfg
        if not c.enforce_budget or c.gpu_budget <= 0:
            return True
        return c.static_bytes + self.resident + extra <= c.gpu_budget

    def _alloc(self, tids, when):
        for tid in tids:
            self.resident += self.size[tid]
            self.deltas.append((when, self.size[tid]))

    def _release(self, tid, when):
        self.resident -= self.size[tid]
        self.deltas.append((when, -self.size[tid]))

    # channels ---------------------------------------------------------------
    def _launch(self, nid, chan, t0, dur):
        heapq.heappush(self.inflight, (t0 + dur, _PRIO[chan], nid, chan))
        self.idle[chan] = False
        self.busy_t[chan] += dur
        self.events.append((nid, chan, t0, t0 + dur))

    def _try_compute(self, now) -> bool:
        if not self.idle["compute"] or self.next_compute >= len(self.serial):
            return False
        nid = self.serial[self.next_compute]
        if self.waits[nid]:
            return False
        node = self.g.node(nid)
        need = sum(self.size[t] for t in node.outputs)
        if not self._fits(need):
            self.budget_blocked = True
            return False
        if now > self.compute_free_at:
            cause = "budget" if self.budget_blocked else self.last_dep.get(nid, (0.0, ""))[1]
            self.stalls.append((nid, cause, now - self.compute_free_at))
        self._alloc(node.outputs, now)
        self._launch(nid, "compute", now, op_cost(node, self.cfg))
        self.next_compute += 1
        self.budget_blocked = False
        return True

    def _try_d2h(self, now) -> bool:
        if not self.idle["d2h"] or not self.d2h_q or self.d2h_q[0][0] > now:
            return False
        nid = heapq.heappop(self.d2h_q)[2]
        nbytes = self.size[self.g.node(nid).inputs[0]]
        self._launch(nid, "d2h", now, xfer_cost(nbytes, self.cfg.d2h_bw, self.cfg.xfer_latency))
        return True

    def _try_h2d(self, now) -> bool:
        if not self.idle["h2d"] or not self.h2d_q:
            return False
        nid = self.h2d_q[0][2]
        if self.waits[nid]:          # head-of-line: its swap_out is still in flight
            return False
        node = self.g.node(nid)
        need = sum(self.size[t] for t in node.outputs)
        if not self._fits(need):
            self.budget_blocked = True
            return False
        heapq.heappop(self.h2d_q)
        self._alloc(node.outputs, now)
        self._launch(nid, "h2d", now, xfer_cost(need, self.cfg.h2d_bw, self.cfg.xfer_latency))
        return True

    def _pump(self, now):
        while True:
            progressed = self._try_compute(now)
            progressed = self._try_d2h(now) or progressed
            progressed = self._try_h2d(now) or progressed
            if not progressed:
                return

    def _complete(self, end, nid, chan):
        g = self.g
        node = g.node(nid)
        self.idle[chan] = True
        if chan == "compute":
            self.compute_free_at = end
        for tid in node.inputs:
            self.readers_left[tid] -= 1
            if not self.readers_left[tid]:
                self._release(tid, end)
        for tid in node.outputs:
            if not self.readers_left[tid]:
                self._release(tid, end)
        for m in sorted(self.succ[nid]):
            self.waits[m] -= 1
            prev = self.last_dep.get(m)
            if prev is None or (end, nid) > prev:
                self.last_dep[m] = (end, nid)
            kind = g.node(m).kind
            if kind == "swap_out" and not self.waits[m]:
                heapq.heappush(self.d2h_q, (end, self.queue_pos[m], m))
            elif kind == "swap_in" and node.kind != "swap_out":
                self.trigger_waits[m] -= 1
                if not self.trigger_waits[m]:
                    heapq.heappush(self.h2d_q, (end, self.queue_pos[m], m))

    def run(self) -> SimReport:
        g, cfg = self.g, self.cfg
        if cfg.enforce_budget and cfg.gpu_budget > 0:
            for t in g.tensors:
                if cfg.static_bytes + self.size[t.id] > cfg.gpu_budget:
                    raise InfeasibleError(t.id, self.size[t.id], cfg.gpu_budget)
        for n in g.nodes:
            if n.kind == "swap_out" and not self.waits[n.id]:
                heapq.heappush(self.d2h_q, (0.0, self.queue_pos[n.id], n.id))
            elif n.kind == "swap_in" and not self.trigger_waits[n.id]:
                heapq.heappush(self.h2d_q, (0.0, self.queue_pos[n.id], n.id))
        done = 0
        self._pump(0.0)
        while done < len(g.nodes):
            if not self.inflight:
                waiting = sorted(set(self.serial[self.next_compute:self.next_compute + 1])
                                 | {q[2] for q in self.d2h_q} | {q[2] for q in self.h2d_q})
                raise DeadlockError(waiting, "budget wait with nothing in flight to free"
                                    if self.budget_blocked else "unsatisfiable dependencies")
            now = self.inflight[0][0]
            while self.inflight and self.inflight[0][0] == now:
                end, _, nid, chan = heapq.heappop(self.inflight)
                done += 1
                self._complete(end, nid, chan)
            self._pump(now)
        makespan = max((e[3] for e in self.events), default=0.0)
        self.events.sort(key=lambda e: (e[2], _PRIO[e[1]], e[0]))
        busy = {c: (self.busy_t[c] / makespan if makespan > 0 else 0.0) for c in CHANNELS}
        return SimReport(makespan=makespan, events=self.events,
                         peak_resident=peak_from_deltas(self.deltas) + cfg.static_bytes,
                         stalls=self.stalls, busy=busy,
                         phases={n.id: n.phase for n in g.nodes})


def simulate(tg: TrainingGraph, plan=None, cfg: SimConfig | None = None) -> SimReport:
    cfg = cfg or SimConfig()
    cfg.validate()
    return _Timeline(tg, cfg).run()


def stall_report(r: SimReport) -> dict[str, float]:
    """Compute-channel idle time split by phase: forward, boundary, backward."""
    first_bw = next((nid for nid, ch, _, _ in r.events
                     if ch == "compute" and r.phases.get(nid) == "backward"), None)
    out = {"forward": 0.0, "boundary": 0.0, "backward": 0.0}
    for nid, _, dur in r.stalls:
        if nid == first_bw:
            out["boundary"] += dur
        elif r.phases.get(nid, "forward") == "backward":
            out["backward"] += dur
        else:
            out["forward"] += dur
    return out


def emit_trace(r: SimReport, path) -> None:
    """Chrome trace ("X" events, tid 0 compute / 1 D2H / 2 H2D, microseconds)."""
    evs = [{"name": nid, "ph": "X", "ts": s * 1e6, "dur": (e - s) * 1e6, "pid": 0,
            "tid": TRACE_TIDS[ch]} for nid, ch, s, e in r.events]
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(evs, sort_keys=True, indent=2) + "\n")


def epoch_time(iter_seconds: float, iterations: int, host_preproc_seconds: float = 0.0) -> float:
    if iterations < 1:
        raise GraphError(f"iterations must be >= 1, got {iterations}")
    return iterations * max(iter_seconds, host_preproc_seconds)


def sweep(tg: TrainingGraph, rewrite_cfgs, sim_cfgs) -> list[dict]:
    from .rewrite import apply_rewrite
    rcfgs, scfgs = list(rewrite_cfgs), list(sim_cfgs)
    if not rcfgs or not scfgs:
        raise GraphError("sweep grid is empty")
    keyed = []
    for rc in rcfgs:
        rw, plan = apply_rewrite(tg, rc)
        for sc in scfgs:
            row = {"n_tensors": rc.n_tensors, "lb": rc.lb, "mode": rc.mode,
                   "d2h_bw": sc.d2h_bw, "h2d_bw": sc.h2d_bw, "swapped": len(plan.swapped)}
            try:
                rep = simulate(rw, plan, sc)
                st = stall_report(rep)
                row.update(makespan=rep.makespan, peak_resident=rep.peak_resident,
                           boundary_stall=st["boundary"], backward_stall=st["backward"],
                           error="")
            except GraphError as exc:
                row.update(makespan=None, peak_resident=None, boundary_stall=None,
                           backward_stall=None, error=str(exc))
            keyed.append(((rc.n_tensors, rc.lb, rc.mode, sc.d2h_bw, sc.h2d_bw), row))
    keyed.sort(key=lambda kr: kr[0])
    return [row for _, row in keyed]


def calibrate_compute_rate(tg: TrainingGraph, plan, cfg: SimConfig, target_makespan: float,
                           tol: float = 1e-3) -> float:
    """Geometric bisection for the compute rate giving ``target_makespan``."""
    if target_makespan <= 0:
        raise GraphError("target makespan must be positive")

    def span(rate):
        c = SimConfig(compute_rate=rate, d2h_bw=cfg.d2h_bw, h2d_bw=cfg.h2d_bw,
                      xfer_latency=cfg.xfer_latency, gpu_budget=cfg.gpu_budget,
                      static_bytes=cfg.static_bytes, enforce_budget=cfg.enforce_budget)
        return simulate(tg, plan, c).makespan

    lo = hi = 1.0
    while span(hi) > target_makespan:
        hi *= 4.0
        if hi > 1e30:
            raise GraphError("target makespan unreachable: transfers alone exceed it")
    while span(lo) < target_makespan:
        lo /= 4.0
        if lo < 1e-30:
            raise GraphError("target makespan unreachable at any compute rate")
    for _ in range(80):
        mid = (lo * hi) ** 0.5
        if span(mid) > target_makespan:
            lo = mid
        else:
            hi = mid
        if hi / lo < 1 + tol:
            break
    return (lo * hi) ** 0.5
