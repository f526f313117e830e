"""GPU: the swap engine executing the reference's toy semantics through the C ABI
must reproduce the reference's run_numeric bit-for-bit (gradients) / to 1e-13
(loss, whose reference value comes from BLAS ddot), and reject broken plans."""
import os

import numpy as np
import pytest

from paper_1812_07816_b200 import numeric
from paper_1812_07816_b200.models import UNetParams, gen_chain, gen_unet3d
from paper_1812_07816_b200.rewrite import PRESETS, RewriteConfig, apply_rewrite, resolve_preset
from paper_1812_07816_b200.training import expand_training_graph

from golden_configs import GOLDEN, build, load

pytestmark = pytest.mark.gpu
INDEX = load("numeric_index.json")


@pytest.mark.parametrize("row", INDEX, ids=lambda r: f"{r['graph']}-{r['preset']}-s{r['seed']}")
def test_gpu_matches_reference_fixture(row):
    tg = expand_training_graph(build(row["graph"]))
    plan = None
    if row["preset"]:
        tg, plan = apply_rewrite(tg, resolve_preset(row["preset"]))
    loss, grads = numeric.run_numeric(tg, plan, row["seed"])
    gold = np.load(os.path.join(GOLDEN, row["file"]))
    ref_loss = float(gold["loss"])
    assert abs(loss - ref_loss) <= 1e-13 * abs(ref_loss)
    for tid in row["grads"]:
        assert np.array_equal(grads[tid], gold[tid.replace(":", "__")]), tid
    if plan is not None:
        st = numeric.last_step_stats()
        swapped = sum(8 * int(np.prod(tg.graph.tensor(t).shape)) * tg.graph.tensor(t).channels
                      for t in plan.swapped)
        assert st["d2h_bytes"] == swapped == st["h2d_bytes"]


def test_gpu_matches_oracle_on_new_sizes():
    from oracle.toy_numeric import run_numeric as oracle_run
    tg = expand_training_graph(gen_unet3d(UNetParams(dims=(16, 16, 16), in_channels=2,
                                                     base_filters=4, depth=3)))
    for preset in (None, "paper-c2", "paper-c4"):
        rw, plan = (tg, None) if preset is None else apply_rewrite(tg, resolve_preset(preset))
        loss, grads = numeric.run_numeric(rw, plan, 11)
        r_loss, r_grads = oracle_run(rw, plan, 11)
        assert abs(loss - r_loss) <= 1e-13 * abs(r_loss)
        assert np.array_equal(grads["source:0"], r_grads["source:0"])


def test_equivalence_all_presets_and_recompute_bit_identical():
    tg = expand_training_graph(gen_unet3d(UNetParams(dims=(8, 8, 8), in_channels=1,
                                                     base_filters=1, depth=2,
                                                     convs_per_level=1)))
    variants = [(p,) + apply_rewrite(tg, resolve_preset(p)) for p in sorted(PRESETS)]
    for policy in ("speed", "sqrt_n"):
        variants.append((f"rc-{policy}",) + apply_rewrite(
            tg, RewriteConfig(mode="recompute", ckpt_policy=policy)))
    rows = numeric.equivalence_check(tg, variants, seeds=[1, 2, 3])
    assert all(r["deviation"] == 0.0 and not r["error"] for r in rows), rows


def test_broken_plan_raises_use_after_swap():
    from paper_1812_07816_b200.graph import GraphSpec
    from paper_1812_07816_b200.training import TrainingGraph
    tg = expand_training_graph(gen_chain(3, bytes_per_tensor=64))
    rw, plan = apply_rewrite(tg, resolve_preset("paper-c1"))
    victim = sorted(plan.swapped)[0]
    in_id = plan.swapped[victim][1]
    g = rw.graph
    in_t = g.node(in_id).outputs[0]
    from paper_1812_07816_b200.graph import NodeSpec
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
    with pytest.raises(numeric.UseAfterSwapError, match="use-after-swap"):
        numeric.run_numeric(broken, plan, 1)


def test_timeline_channels_and_stalls():
    tg = expand_training_graph(gen_unet3d(UNetParams(dims=(32, 32, 32), in_channels=4,
                                                     base_filters=8, depth=3)))
    rw, plan = apply_rewrite(tg, resolve_preset("paper-c1"))
    numeric.run_numeric(rw, plan, 1)
    eng = numeric._engine
    tl = eng.timeline()
    chans = {c for _, c, _, _ in tl}
    assert {0, 1, 2} <= chans
    n_d2h = sum(1 for _, c, _, _ in tl if c == 1)
    assert n_d2h == len(plan.swapped)
    for _, c, s, e in tl:
        assert e >= s >= 0.0


class TestGradCheckOnGpu:
    """grad_check drop-in (reference numeric.py:361-400, tests test_numeric.py:53-74): the
    GPU step's analytic gradients against central differences of the GPU forward loss."""

    @staticmethod
    def chain(n, kinds=("conv",)):
        return expand_training_graph(gen_chain(n, bytes_per_tensor=64, kinds=kinds))

    def test_chain3(self):
        rep = numeric.grad_check(self.chain(3, ("conv", "activation", "norm")), seed=0,
                                 eps=1e-5)
        assert rep.max_rel_error < 1e-4

    def test_single_affine_node_is_nearly_exact(self):
        assert numeric.grad_check(self.chain(1), seed=0, eps=1e-5).max_rel_error < 1e-7

    def test_unet_toy(self):
        tg = expand_training_graph(gen_unet3d(UNetParams(dims=(8, 8, 8), in_channels=1,
                                                         base_filters=1, depth=2,
                                                         convs_per_level=1)))
        assert numeric.grad_check(tg, seed=1, eps=1e-5).max_rel_error < 1e-4

    def test_zero_input_at_activation_kink_is_resampled(self):
        tg = self.chain(2, ("conv", "activation"))
        rep = numeric.grad_check(tg, seed=0, inputs={"t0": np.zeros(64)})
        assert rep.resampled and rep.seed_used != 0
        assert rep.max_rel_error < 1e-4

    def test_bad_eps_is_a_domain_error(self):
        from paper_1812_07816_b200.graph import GraphError
        with pytest.raises(GraphError):
            numeric.grad_check(self.chain(1), eps=0.0)


def test_budget_failures_raise_the_reference_exception_types():
    """An arena too small for one tensor is InfeasibleError; one whose bytes are all held
    by live tensors is DeadlockError (reference sim.py:33-43)."""
    from paper_1812_07816_b200.sim import DeadlockError, InfeasibleError
    from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer
    base = dict(dims=(32, 32, 32), base_filters=16, depth=3, dtype="bf16", preset=None)
    with pytest.raises(InfeasibleError):
        tr = UNetTrainer(TrainConfig(arena_bytes=512 << 10, **base))
        tr.step(*tr.synthetic_batch())
    probe = UNetTrainer(TrainConfig(**base), device_engine=False)
    with pytest.raises(DeadlockError):
        tr = UNetTrainer(TrainConfig(arena_bytes=probe.program.order_peak() // 2, **base))
        tr.step(*tr.synthetic_batch())
