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
