"""Timeline-model parity with the reference simulator (golden sim.json)."""
import hashlib

import pytest

from paper_1812_07816_b200.graph import GraphError
from paper_1812_07816_b200.rewrite import apply_rewrite, resolve_preset
from paper_1812_07816_b200.sim import SimConfig, simulate, stall_report
from paper_1812_07816_b200.training import expand_training_graph

from golden_configs import build, load

CASES = load("sim.json")


@pytest.mark.parametrize("row", CASES, ids=lambda r: f"{r['graph']}-{r['preset']}")
def test_simulate_matches_reference(row):
    tg = expand_training_graph(build(row["graph"]))
    plan = None
    if row["preset"]:
        tg, plan = apply_rewrite(tg, resolve_preset(row["preset"]))
    if row["error"]:
        with pytest.raises(GraphError) as ei:
            simulate(tg, plan, SimConfig(**row["sim"]))
        assert type(ei.value).__name__ + ": " + str(ei.value) == row["error"]
        return
    rep = simulate(tg, plan, SimConfig(**row["sim"]))
    if "report_json" in row:
        assert rep.to_json() == row["report_json"]
    assert hashlib.sha256(rep.to_json().encode()).hexdigest() == row["report_sha"]
    assert rep.makespan == row["makespan"]
    assert rep.peak_resident == row["peak_resident"]
    assert stall_report(rep) == row["stall"]


def test_stall_accounting_identity():
    from paper_1812_07816_b200.models import gen_chain
    tg = expand_training_graph(gen_chain(6, bytes_per_tensor=5000, cost_per_op=2.0))
    rw, plan = apply_rewrite(tg, resolve_preset("paper-c1"))
    r = simulate(rw, plan, SimConfig(compute_rate=1.0, d2h_bw=900.0, h2d_bw=700.0))
    busy = sum(e - s for _, ch, s, e in r.events if ch == "compute")
    assert busy + sum(d for _, _, d in r.stalls) == pytest.approx(r.makespan)
