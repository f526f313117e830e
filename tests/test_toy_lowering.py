"""The toy-mode program the GPU runs, interpreted on the CPU by tests/mock_engine.py,
must reproduce the reference run_numeric() bit-for-bit (golden numeric_*.npz), and
a plan with a deleted swap_in must be rejected as a use-after-swap."""
import os

import numpy as np
import pytest

from paper_1812_07816_b200.lowering import lower_toy
from paper_1812_07816_b200.models import UNetParams, gen_chain, gen_unet3d
from paper_1812_07816_b200.rewrite import RewriteConfig, apply_rewrite, resolve_preset
from paper_1812_07816_b200.training import expand_training_graph

from golden_configs import GOLDEN, build, load
from mock_engine import MockUseAfterSwap, run_program

INDEX = load("numeric_index.json")


def _case(gname, preset):
    tg = expand_training_graph(build(gname))
    plan = None
    if preset:
        tg, plan = apply_rewrite(tg, resolve_preset(preset))
    return tg, plan


def run_mock(tg, plan, seed):
    low = lower_toy(tg, plan, seed)
    persist, stats = run_program(low.program, {s: v for s, v in low.inputs.values()})
    loss = float(persist[low.loss_tid][0])
    grads = {t: persist[r] for t, r in low.results.items()}
    return loss, grads, stats


@pytest.mark.parametrize("row", INDEX, ids=lambda r: f"{r['graph']}-{r['preset']}-s{r['seed']}")
def test_mock_program_matches_reference(row):
    tg, plan = _case(row["graph"], row["preset"])
    loss, grads, _ = run_mock(tg, plan, row["seed"])
    gold = np.load(os.path.join(GOLDEN, row["file"]))
    assert loss == float(gold["loss"])
    for tid in row["grads"]:
        assert np.array_equal(grads[tid], gold[tid.replace(":", "__")]), tid


def test_swap_traffic_matches_plan():
    tg, plan = _case("toy8", "paper-c1")
    _, _, stats = run_mock(tg, plan, 1)
    expected = sum(8 * np.prod(tg.graph.tensor(t).shape) * tg.graph.tensor(t).channels
                   for t in plan.swapped)
    assert stats["d2h"] == expected == stats["h2d"]


def test_recompute_plans_run_on_the_program_path():
    tg = expand_training_graph(gen_chain(9, bytes_per_tensor=64,
                                         kinds=("conv", "activation", "norm")))
    base = run_mock(tg, None, 4)
    for policy in ("speed", "sqrt_n"):
        rw, plan = apply_rewrite(tg, RewriteConfig(mode="recompute", ckpt_policy=policy))
        got = run_mock(rw, plan, 4)
        assert got[0] == base[0]
        assert np.array_equal(got[1]["t0"], base[1]["t0"])


def test_broken_plan_is_use_after_swap():
    from paper_1812_07816_b200.graph import GraphSpec, NodeSpec
    from paper_1812_07816_b200.training import TrainingGraph
    tg = expand_training_graph(gen_chain(3, bytes_per_tensor=64))
    rw, plan = apply_rewrite(tg, resolve_preset("paper-c1"))
    victim = sorted(plan.swapped)[0]
    in_id = plan.swapped[victim][1]
    g = rw.graph
    in_t = g.node(in_id).outputs[0]
    nodes = tuple(NodeSpec(id=n.id, kind=n.kind,
                           inputs=tuple(victim if t == in_t else t for t in n.inputs),
                           outputs=n.outputs, cost_units=n.cost_units, scope=n.scope,
                           phase=n.phase) for n in g.nodes if n.id != in_id)
    broken = TrainingGraph(graph=GraphSpec(nodes=nodes,
                                           tensors=tuple(t for t in g.tensors if t.id != in_t),
                                           control_edges=tuple(e for e in g.control_edges
                                                               if in_id not in e),
                                           metadata=dict(g.metadata)),
                           reuse_edges=rw.reuse_edges, serial_order=rw.serial_order,
                           grad_of=dict(rw.grad_of))
    with pytest.raises(MockUseAfterSwap, match="use-after-swap"):
        run_mock(broken, plan, 1)


def test_unet_toy_all_presets_deviation_zero():
    tg = expand_training_graph(gen_unet3d(UNetParams(dims=(8, 8, 8), in_channels=1,
                                                     base_filters=1, depth=2,
                                                     convs_per_level=1)))
    base = run_mock(tg, None, 7)
    for p in ("paper-c1", "paper-c2", "paper-c3", "paper-c4"):
        rw, plan = apply_rewrite(tg, resolve_preset(p))
        got = run_mock(rw, plan, 7)
        assert got[0] == base[0]
        assert np.array_equal(got[1]["source:0"], base[1]["source:0"])
