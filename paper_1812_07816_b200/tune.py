"""Calibrated swap-plan tuner.

The reference ships a discrete-event model of the step (``simulate``,
sim.py:114) and a sweep over rewrite configurations (``sweep``,
sim.py:351-382), but calibrates it with one scalar compute rate
(``calibrate_compute_rate``, sim.py:385-415).  On the B200 the step is far
from uniform (tensor-core convs vs HBM-bound norms), so this module feeds the
model the *measured* per-slot compute times of a real step and the *measured*
host-link bandwidths, then searches the planner's knobs -- ``n_tensors`` (the
count threshold), ``lb`` and the scope filters -- for the plan with the
smallest predicted step time whose static peak fits an HBM budget.  The
result is an ordinary ``RewriteConfig``, so the chosen plan is still produced
by the byte-exact planner and executed byte-for-byte by the engine.
"""
from __future__ import annotations

from dataclasses import dataclass

from .graph import GraphSpec, NodeSpec
from .rewrite import RewriteConfig, apply_rewrite
from .sim import SimConfig, simulate, stall_report
from .training import TrainingGraph, static_peak_estimate


def with_measured_costs(tg: TrainingGraph, slot_seconds: dict) -> TrainingGraph:
    """Copy of tg whose compute nodes cost their measured seconds (compute_rate 1)."""
    g = tg.graph
    nodes = tuple(NodeSpec(id=n.id, kind=n.kind, inputs=n.inputs, outputs=n.outputs,
                           cost_units=0.0 if n.phase == "io" else float(slot_seconds.get(n.id, 0.0)),
                           scope=n.scope, phase=n.phase) for n in g.nodes)
    return TrainingGraph(graph=GraphSpec(nodes=nodes, tensors=g.tensors,
                                         control_edges=g.control_edges, metadata=g.metadata),
                         reuse_edges=tg.reuse_edges, serial_order=tg.serial_order,
                         grad_of=dict(tg.grad_of))


@dataclass
class TuneResult:
    config: RewriteConfig
    makespan: float
    exposed: float          # (makespan - compute) / makespan
    peak_bytes: int
    swapped: int
    swapped_bytes: int
    stalls: dict


def predict(tg: TrainingGraph, cfg: RewriteConfig, slot_seconds: dict, d2h_bw: float,
            h2d_bw: float) -> TuneResult:
    rw, plan = apply_rewrite(tg, cfg)
    cal = with_measured_costs(rw, slot_seconds)
    rep = simulate(cal, plan, SimConfig(compute_rate=1.0, d2h_bw=d2h_bw, h2d_bw=h2d_bw))
    compute = sum(e - s for _, ch, s, e in rep.events if ch == "compute")
    from .graph import tensor_bytes
    nbytes = sum(tensor_bytes(rw.graph.tensor(t)) for t in plan.swapped)
    return TuneResult(config=cfg, makespan=rep.makespan,
                      exposed=(rep.makespan - compute) / rep.makespan if rep.makespan else 0.0,
                      peak_bytes=static_peak_estimate(rw, plan).peak_bytes,
                      swapped=len(plan.swapped), swapped_bytes=nbytes,
                      stalls=stall_report(rep))


def autotune(tg: TrainingGraph, slot_seconds: dict, d2h_bw: float, h2d_bw: float,
             budget_bytes: int | None = None, max_exposed: float | None = None,
             lbs=(1, 5, 10, 20, 40, 73, 1000), scope_sets=None) -> list[TuneResult]:
    """Rank swap configurations by predicted step time (peak within budget).

    With ``max_exposed`` set, the fastest plan swapping the MOST bytes while
    staying under that exposed fraction is ranked first (the paper's goal:
    relieve as much memory as the link can hide)."""
    from .training import cross_phase_tensors
    n_cand = len(cross_phase_tensors(tg))
    scope_sets = scope_sets or [((), ()), (("synthesis/*",), ())]
    results = []
    for excl, incl in scope_sets:
        for n in range(1, n_cand + 1):
            for lb in lbs:
                cfg = RewriteConfig(mode="swap", n_tensors=n, lb=lb, excl_scopes=tuple(excl),
                                    incl_scopes=tuple(incl))
                r = predict(tg, cfg, slot_seconds, d2h_bw, h2d_bw)
                if budget_bytes is not None and r.peak_bytes > budget_bytes:
                    continue
                results.append(r)
    if max_exposed is not None:
        ok = [r for r in results if r.exposed <= max_exposed]
        rest = [r for r in results if r.exposed > max_exposed]
        ok.sort(key=lambda r: (-r.swapped_bytes, r.makespan))
        rest.sort(key=lambda r: r.makespan)
        return ok + rest
    results.sort(key=lambda r: (r.makespan, -r.swapped_bytes))
    return results
