"""Train-step API on the GPU: the drop-in for ``run_numeric`` and friends.

``run_numeric(tg, plan=None, seed=0, inputs=None) -> (loss, {input: grad})``
keeps the reference signature and semantics (pkg/src/swapsim/numeric.py:153)
but executes on the B200 through libunetswap: the graph is lowered to a
device program (``lowering.lower_toy``) and the swap engine moves every
planned tensor to pinned host memory and back on its copy streams.  The toy
arithmetic is reproduced bit-for-bit (numpy summation order), so results
equal the reference's; residency violations surface as the same
``UseAfterSwapError``.  There is no host fallback: without the CUDA library
or a GPU these functions raise.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._native import US_ERR_DOMAIN, Engine, EngineError
from .graph import GraphError, element_count
from .lowering import lower_toy
from .training import TrainingGraph

MAX_ELEMENTS = 1 << 26   # the device executor is not capped at the reference's 10k elements
KINK_TOL = 1e-6          # reference numeric.py:26


class UseAfterSwapError(GraphError):
    def __init__(self, message: str, tensor_id: str = ""):
        super().__init__(message)
        self.tensor_id = tensor_id


_engine = None


def _get_engine(arena_bytes: int) -> Engine:
    global _engine
    if _engine is None or _engine.arena_bytes < arena_bytes:
        if _engine is not None:
            _engine.close()
        _engine = Engine(0, max(arena_bytes, 64 << 20))
    return _engine


def _raise_domain(exc: EngineError):
    msg = str(exc)
    if exc.code == US_ERR_DOMAIN and "use-after-swap" in msg:
        tid = ""
        if "tensor '" in msg:
            tid = msg.split("tensor '", 1)[1].split("'", 1)[0]
        raise UseAfterSwapError(msg, tid) from None
    if exc.code == US_ERR_DOMAIN and "budget exhausted" in msg:
        # the engine's arena failures carry the reference's exception types (sim.py:33-43)
        from .sim import DeadlockError, InfeasibleError
        tid = msg.split("tensor '", 1)[1].split("'", 1)[0] if "tensor '" in msg else ""
        if "infeasible:" in msg:
            nums = [int(w) for w in msg.replace(",", " ").split() if w.isdigit()]
            err = InfeasibleError(tid, nums[0] if nums else 0, nums[1] if len(nums) > 1 else 0)
        else:
            err = DeadlockError([tid], msg)
        err.engine_message = msg
        raise err from None
    if exc.code == US_ERR_DOMAIN:
        raise GraphError(msg) from None
    raise exc


def _check_sizes(g) -> None:
    for t in g.tensors:
        if element_count(t) > MAX_ELEMENTS:
            raise GraphError(f"tensor {t.id!r} has {element_count(t)} elements; the numeric "
                             f"executor is capped at {MAX_ELEMENTS}")


def run_numeric(tg: TrainingGraph, plan=None, seed: int = 0,
                inputs=None) -> tuple[float, dict[str, np.ndarray]]:
    """Execute the training graph on the GPU; returns (loss, per-input gradients)."""
    _check_sizes(tg.graph)
    low = lower_toy(tg, plan, seed, inputs)
    eng = _get_engine(low.program.arena_need())
    try:
        low.program.emit(eng)
        for staging, values in low.inputs.values():
            eng.upload(staging, values)
        eng.run()
        eng.sync()
    except EngineError as exc:
        _raise_domain(exc)
    loss = float(eng.download(low.loss_tid, 8, np.float64)[0])
    grads = {}
    for tid, res in low.results.items():
        nbytes = low.program.by_tid()[res].nbytes
        grads[tid] = eng.download(res, nbytes, np.float64)
    return loss, grads


def last_step_stats() -> dict:
    """Engine counters of the last run_numeric call (swap bytes, arena peak, stalls)."""
    if _engine is None:
        raise GraphError("no step has run")
    return _engine.stats()


def equivalence_check(tg: TrainingGraph, variants, seeds) -> list[dict]:
    """Max |difference| of loss and gradients between each rewritten variant and the
    unrewritten graph (reference numeric.py:403-430), all executed on the GPU."""
    rows = []
    base = {s: run_numeric(tg, None, s) for s in seeds}
    for label, var_tg, plan in variants:
        worst, error = 0.0, ""
        for s in seeds:
            b_loss, b_grads = base[s]
            try:
                loss, grads = run_numeric(var_tg, plan, s)
            except GraphError as exc:
                error, worst = str(exc), float("inf")
                break
            worst = max(worst, abs(loss - b_loss))
            for tid, arr in b_grads.items():
                if tid not in grads:
                    error, worst = f"missing gradient for {tid!r}", float("inf")
                    break
                if arr.size:
                    worst = max(worst, float(np.max(np.abs(arr - grads[tid]))))
            if error:
                break
        rows.append({"label": label, "deviation": worst, "error": error})
    return rows


@dataclass
class GradCheckReport:
    max_rel_error: float
    seed_used: int
    resampled: bool


class _ToyRunner:
    """One lowered + emitted toy program, re-run with new input values (grad_check)."""

    def __init__(self, tg: TrainingGraph, point: dict):
        from .lowering import lower_toy
        self.low = lower_toy(tg, None, 0, inputs=point, capture_activation_inputs=True)
        self.eng = _get_engine(self.low.program.arena_need())
        self.defs = self.low.program.by_tid()
        try:
            self.low.program.emit(self.eng)
        except EngineError as exc:
            _raise_domain(exc)

    def run(self, point: dict, grads: bool = False):
        eng = self.eng
        try:
            for tid, (staging, _) in self.low.inputs.items():
                eng.upload(staging, np.asarray(point[tid], np.float64))
            eng.run()
            eng.sync()
        except EngineError as exc:
            _raise_domain(exc)
        loss = float(eng.download(self.low.loss_tid, 8, np.float64)[0])
        if not grads:
            return loss, None
        return loss, {tid: eng.download(res, self.defs[res].nbytes, np.float64)
                      for tid, res in self.low.results.items()}

    def kink_distance(self, point: dict) -> float:
        """Smallest |activation input| of a forward pass at ``point`` (numeric.py:325)."""
        self.run(point)
        closest = float("inf")
        for tid in self.low.act_inputs.values():
            v = self.eng.download(tid, self.defs[tid].nbytes, np.float64)
            if v.size:
                closest = min(closest, float(np.abs(v).min()))
        return closest


def grad_check(tg: TrainingGraph, seed: int = 0, eps: float = 1e-5,
               inputs=None) -> GradCheckReport:
    """Max relative error between the GPU step's analytic gradients and central
    differences of the GPU forward loss (reference numeric.py:361-400, same signature,
    resampling rule and report).  Sample points that land an activation input on its
    kink are resampled with seed + 101 (``resampled`` / ``seed_used``)."""
    from .lowering import input_values
    if eps <= 0:
        raise GraphError("eps must be positive")
    g = tg.graph
    _check_sizes(g)
    seed_used, resampled = seed, False
    point = dict(input_values(g, seed, inputs))
    runner = _ToyRunner(tg, point)
    for _ in range(16):
        if runner.kink_distance(point) > max(KINK_TOL, 2 * eps):
            break
        resampled = True
        seed_used += 101
        point = dict(input_values(g, seed_used, None))
    _, analytic = runner.run(point, grads=True)
    worst = 0.0
    for tid, garr in sorted(analytic.items()):
        base = point[tid]
        for j in range(base.size):
            bumped = dict(point)
            plus = base.copy()
            plus[j] += eps
            minus = base.copy()
            minus[j] -= eps
            bumped[tid] = plus
            lp, _ = runner.run(bumped)
            bumped[tid] = minus
            lm, _ = runner.run(bumped)
            num = (lp - lm) / (2 * eps)
            denom = max(abs(garr[j]), abs(num), 1e-12)
            worst = max(worst, abs(garr[j] - num) / denom)
    if not np.isfinite(worst):
        raise GraphError("gradient check produced non-finite values")
    return GradCheckReport(max_rel_error=worst, seed_used=seed_used, resampled=resampled)
