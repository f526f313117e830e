"""Planner parity: this package's model builder / expansion / swap planner must
reproduce the reference's artifacts byte-for-byte (golden fixtures made by
tests/golden/make_golden.py from the unmodified reference)."""
import hashlib

import pytest

from paper_1812_07816_b200.graph import dumps_canonical, graph_to_obj
from paper_1812_07816_b200.rewrite import RewriteConfig, apply_rewrite, select_swap_tensors
from paper_1812_07816_b200.training import (cross_phase_tensors, expand_training_graph,
                                            static_peak_estimate, training_to_obj)

from golden_configs import build, load

GOLD = load("planner.json")


def sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


@pytest.fixture(scope="module")
def expanded():
    cache = {}

    def get(name):
        if name not in cache:
            g = build(name)
            cache[name] = (g, expand_training_graph(g))
        return cache[name]
    return get


@pytest.mark.parametrize("name", sorted(GOLD))
def test_graph_and_expansion_bytes(name, expanded):
    g, tg = expanded(name)
    rec = GOLD[name]
    assert (len(g.nodes), len(g.tensors)) == (rec["n_nodes"], rec["n_tensors"])
    assert sha(dumps_canonical(graph_to_obj(g))) == rec["forward_sha"]
    assert list(tg.serial_order) == rec["serial_order"]
    assert sha(dumps_canonical(training_to_obj(tg))) == rec["training_sha"]
    assert cross_phase_tensors(tg) == rec["cross_phase"]
    assert static_peak_estimate(tg).peak_bytes == rec["noswap_peak"]


def _cases():
    for name in sorted(GOLD):
        for case in GOLD[name]["cases"]:
            yield pytest.param(name, case, id=f"{name}-{case['label']}")


@pytest.mark.parametrize("name,case", list(_cases()))
def test_plan_bytes(name, case, expanded):
    _, tg = expanded(name)
    kw = dict(case["cfg"])
    mode = kw.pop("mode", "swap")
    for k in ("excl_scopes", "incl_scopes"):
        if k in kw:
            kw[k] = tuple(kw[k])
    cfg = RewriteConfig(mode=mode, **kw)
    if mode == "swap":
        assert select_swap_tensors(tg, cfg) == case["selection"]
    rw, plan = apply_rewrite(tg, cfg)
    pj = plan.to_json()
    if "plan_json" in case:
        assert pj == case["plan_json"]
    assert sha(pj) == case["plan_sha"]
    assert sha(dumps_canonical(training_to_obj(rw))) == case["rewritten_sha"]
    rep = static_peak_estimate(rw, plan)
    assert rep.peak_bytes == case["peak"]
    if "peak_position" in case:
        assert rep.peak_position == case["peak_position"]


def test_paper_table_counts(expanded):
    # Acceptance criterion 4 of the reference (test_acceptance.py:126-146): (73, 73, 41, 41).
    from paper_1812_07816_b200.rewrite import resolve_preset
    _, tg = expanded("f192")
    counts = tuple(len(apply_rewrite(tg, resolve_preset(p))[1].swapped)
                   for p in ("paper-c1", "paper-c2", "paper-c3", "paper-c4"))
    assert counts == (73, 73, 41, 41)


def test_plan_is_size_independent(expanded):
    # the plan depends only on topology + config.
    from paper_1812_07816_b200.rewrite import resolve_preset
    shas = {sha(apply_rewrite(expanded(n)[1], resolve_preset("paper-c4"))[1].to_json())
            for n in ("p128", "f192", "f192_bf16", "n240")}
    assert len(shas) == 1
