"""Calibrated plan tuner: uses the reference timeline model with measured costs."""
import pytest

from paper_1812_07816_b200.models import UNetParams, gen_unet3d
from paper_1812_07816_b200.rewrite import resolve_preset
from paper_1812_07816_b200.sim import SimConfig, simulate
from paper_1812_07816_b200.training import expand_training_graph, static_peak_estimate
from paper_1812_07816_b200.tune import autotune, predict, with_measured_costs


@pytest.fixture(scope="module")
def tg():
    return expand_training_graph(gen_unet3d(UNetParams(dims=(32, 32, 32), in_channels=4,
                                                       base_filters=8, depth=3, elem_bytes=2)))


def slot_times(tg):
    # synthetic "measured" costs: proportional to the reference cost model
    return {n.id: n.cost_units / 1e12 for n in tg.graph.nodes if n.phase != "io"}


def test_measured_costs_reproduce_compute_sum(tg):
    st = slot_times(tg)
    rep = simulate(with_measured_costs(tg, st), None, SimConfig(compute_rate=1.0))
    assert rep.makespan == pytest.approx(sum(st[n] for n in tg.serial_order))


def test_predict_matches_direct_simulation(tg):
    st = slot_times(tg)
    r = predict(tg, resolve_preset("paper-c4"), st, 1e9, 1e9)
    assert r.swapped == 27
    assert r.makespan > sum(st[n] for n in tg.serial_order) * 0.999


def test_autotune_respects_budget_and_ranks(tg):
    st = slot_times(tg)
    full = static_peak_estimate(tg).peak_bytes
    budget = int(full * 0.8)
    res = autotune(tg, st, 2e9, 2e9, budget_bytes=budget, lbs=(1, 20))
    assert res and all(r.peak_bytes <= budget for r in res)
    spans = [r.makespan for r in res]
    assert spans == sorted(spans)
    ranked = autotune(tg, st, 2e9, 2e9, budget_bytes=budget, max_exposed=0.5, lbs=(1, 20))
    ok = [r for r in ranked if r.exposed <= 0.5]
    if ok:
        assert ranked[0].exposed <= 0.5


# --------------------------------------------------------------- engine-aware tuner

def _small_cfg():
    from paper_1812_07816_b200.unet import TrainConfig
    return TrainConfig(dims=(32, 32, 32), base_filters=8, depth=3, batch=1, preset=None,
                       dtype="bf16")


def test_candidate_modes(tg):
    from paper_1812_07816_b200.tune import candidate_rewrites
    swap = candidate_rewrites(tg, modes="swap")
    every = candidate_rewrites(tg, modes="all")
    assert all(not isinstance(rw, tuple) and rw.mode in ("none", "swap") for _, rw in swap)
    assert any(not isinstance(rw, tuple) and rw.mode == "recompute" for _, rw in every)
    # level whitelists of the analysis path are searched (the reference's incl_scopes)
    incl = {rw.incl_scopes for _, rw in swap if not isinstance(rw, tuple)}
    assert ("analysis/l1/*",) in incl and ("analysis/l0/*", "analysis/l1/*") in incl
    with pytest.raises(ValueError):
        candidate_rewrites(tg, modes="bogus")


def test_tune_for_budget_forces_swapping_below_the_unswapped_peak():
    """A budget the unswapped program cannot be laid out in: every ranked swap-mode plan
    swaps, fits its static layout in the budget, and the unswapped plan is absent."""
    import dataclasses

    from paper_1812_07816_b200.engine_model import estimate_slot_seconds
    from paper_1812_07816_b200.sim import DeadlockError, InfeasibleError
    from paper_1812_07816_b200.tune import tune_for_budget
    from paper_1812_07816_b200.unet import UNetTrainer
    base = _small_cfg()
    probe = UNetTrainer(dataclasses.replace(base, placement="best_fit"), device_engine=False)
    slots = estimate_slot_seconds(probe.rw, {})
    peak = probe.program.order_peak()
    budget = int(peak * 0.9)
    with pytest.raises((DeadlockError, InfeasibleError)):
        UNetTrainer(dataclasses.replace(base, arena_bytes=budget, slot_seconds=slots),
                    device_engine=False)
    ranked = tune_for_budget(base, slots, 50e9, 50e9, budget, modes="swap", shortlist=8)
    assert ranked
    for c in ranked:
        assert c.swapped > 0 and c.recomputed == 0 and c.label != "none"
        assert c.pred.layout_peak <= budget
