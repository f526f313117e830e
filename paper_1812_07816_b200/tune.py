"""Calibrated swap-plan tuner.

Two predictors live here.  ``predict`` / ``autotune`` feed the reference's own
timeline model (sim.py) with measured slot times: they price the *plan*.
``tune_for_budget`` is what the bench uses: it lowers every candidate plan to the
engine program it would really run and prices that program with
``engine_model.predict`` (dead BatchNorm outputs, direct concat, fused ReLU
gradients, workspaces, need-order swap-outs, memory that comes back only when a
swap-out finishes), over swap plans, recompute plans and recompute+swap mixes
(rewrite.apply_rewrites).

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


# ---------------------------------------------------------------------------
# Engine-aware tuning (what the bench runs)

@dataclass
class Candidate:
    label: str
    rewrite: object                 # RewriteConfig or a tuple (rewrite.apply_rewrites)
    pred: object                    # engine_model.Prediction
    swapped: int
    moved_bytes: int                # bytes per direction the engine moves
    recomputed: int                 # recompute clones

    def summary(self) -> dict:
        p = self.pred
        return {"label": self.label, "predicted_ms": 1e3 * p.step_s,
                "predicted_exposed_pct": 100 * p.exposed,
                "predicted_physical_peak_bytes": p.physical_peak,
                "layout_peak_bytes": p.layout_peak,
                "layout_hold_fraction": getattr(p, "hold_fraction", None),
                "swapped_tensors": self.swapped, "moved_bytes_per_direction": self.moved_bytes,
                "recompute_clones": self.recomputed}


TUNE_MODES = ("swap", "all")


def candidate_rewrites(tg: TrainingGraph, elide_dead_norm="unswapped",
                       lbs=(1, 3, 10, 20, 40, 60, 80, 1000), modes: str = "all"):
    """(label, rewrite) pairs: swap plans over n_tensors / lb / scope filters (with and
    without the BatchNorm outputs, which nobody reads back -- only without them when the
    engine skips their planned swaps, so every planned swap is executed), recompute plans,
    and recompute followed by swapping n of the kept checkpoints.

    modes: "all" (swap, recompute and mixed plans) or "swap" (the paper's data swapping
    only: the unswapped plan and the swap plans -- the forced-swap regime)."""
    from .training import cross_phase_tensors
    from .graph import scope_matches
    if modes not in TUNE_MODES:
        raise ValueError(f"modes must be one of {TUNE_MODES}, got {modes!r}")
    norms = [("*/norm*",)] if elide_dead_norm in (True, "all") else [(), ("*/norm*",)]
    out = [("none", RewriteConfig(mode="none"))]
    # scope filters: the paper's (everything / no synthesis) and whitelists of one or two
    # consecutive analysis levels.  The shallowest tensors the unfiltered threshold picks
    # first are the full-resolution ones, needed last in backward and each larger than the
    # link moves during a B200 forward pass; a level whitelist lets the threshold start at a
    # level whose copies the step can hide.
    levels = sorted({n.scope.split("/")[1] for n in tg.graph.nodes
                     if n.scope.startswith("analysis/") and n.scope.count("/") >= 1})
    scope_sets = [((), ()), (("synthesis/*",), ())]
    scope_sets += [((), (f"analysis/{lv}/*",)) for lv in levels]
    scope_sets += [((), (f"analysis/{a}/*", f"analysis/{b}/*")) for a, b in zip(levels, levels[1:])]
    for norm, (extra, incl) in [(nm, ss) for nm in norms for ss in scope_sets]:
        excl = norm + extra
        cands = [t for t in cross_phase_tensors(tg)
                 if (not incl or scope_matches(tg.graph.node(tg.graph.tensor(t).producer).scope,
                                               incl))
                 and not scope_matches(tg.graph.node(tg.graph.tensor(t).producer).scope, excl)]
        for n in range(1, len(cands) + 1):
            for lb in lbs:
                out.append((f"swap n={n} lb={lb} excl={','.join(excl) or '-'}"
                            + (f" incl={','.join(incl)}" if incl else ""),
                            RewriteConfig(mode="swap", n_tensors=n, lb=lb, excl_scopes=excl,
                                          incl_scopes=incl)))
    if modes == "swap":
        return out
    for pol in ("speed", "sqrt_n"):
        rc = RewriteConfig(mode="recompute", ckpt_policy=pol)
        out.append((f"recompute {pol}", rc))
        rw, _ = apply_rewrite(tg, rc)
        n_ck = len(cross_phase_tensors(rw))
        for n in range(1, n_ck + 1):
            for lb in lbs:
                out.append((f"recompute {pol} + swap n={n} lb={lb}",
                            (rc, RewriteConfig(mode="swap", n_tensors=n, lb=lb))))
    return out


def slot_seconds_for(trainer, measured: dict) -> dict:
    """Measured slot times mapped onto a candidate's serial order: a recompute clone costs
    what its original forward op cost."""
    clone_of = dict(trainer.plan.clone_map) if trainer.plan is not None else {}
    out = {}
    for nid in trainer.rw.serial_order:
        out[nid] = measured.get(clone_of.get(nid, nid), measured.get(nid, 0.0))
    out["optimizer"] = measured.get("optimizer", 0.0)
    return out


def tune_for_budget(base_cfg, measured: dict, d2h_bw: float, h2d_bw: float, budget: int,
                    lbs=(1, 3, 10, 20, 40, 60, 80, 1000), shortlist: int = 40,
                    progress=None, modes: str = "all") -> list[Candidate]:
    """Rank candidate plans for an HBM budget by the engine model's predicted step time.

    base_cfg: a unet.TrainConfig (dims, batch, dtype, elide_dead_norm ... ); measured:
    compute seconds per slot name from a timeline step (engine_model
    .slot_times_from_timeline).  Every candidate is lowered to its engine program and
    priced with byte-count memory (engine_model.predict); the ``shortlist`` fastest that
    fit are then given the static arena layout the engine will use (plan_layout: regions
    of swapped-out tensors held until their copies are predicted done, shortened until the
    layout fits the budget) and re-priced with exact region waits.  Returns the
    candidates whose layout fits, fastest first.  modes: see candidate_rewrites."""
    import dataclasses
    from .engine_model import plan_layout
    from .engine_model import predict as engine_predict
    from .unet import UNetTrainer
    probe = UNetTrainer(dataclasses.replace(base_cfg, preset=None, rewrite=None,
                                            placement="best_fit"), device_engine=False)
    seen, first = set(), []
    for label, rw in candidate_rewrites(probe.tg, base_cfg.elide_dead_norm, lbs, modes):
        tr = UNetTrainer(dataclasses.replace(base_cfg, preset=None, rewrite=rw,
                                             placement="best_fit"), device_engine=False)
        key = tr.plan.to_json()
        if key in seen:
            continue
        seen.add(key)
        slots = slot_seconds_for(tr, measured)
        pred = engine_predict(tr.program, slots, d2h_bw, h2d_bw, budget)
        if progress:
            progress(label, pred)
        if pred.feasible:
            first.append((pred.step_s, label, rw, tr, slots))
    first.sort(key=lambda r: r[0])
    out = []
    for _, label, rw, tr, slots in first[:shortlist]:
        offs, peak, frac = plan_layout(tr.program, slots, d2h_bw, h2d_bw, budget)
        if offs is None:
            continue
        pred = engine_predict(tr.program, slots, d2h_bw, h2d_bw, budget, offsets=offs)
        if not pred.feasible:
            continue
        pred.hold_fraction = frac
        out.append(Candidate(label, rw, pred, len(tr.plan.swapped), pred.d2h_bytes,
                             len(tr.plan.clone_map)))
    out.sort(key=lambda c: (c.pred.step_s, c.moved_bytes))
    return out
