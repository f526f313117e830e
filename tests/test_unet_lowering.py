"""CPU checks of the real-op lowering (no GPU): the program the engine runs must be
residency-sound, move exactly the plan's bytes, and read every prefetched tensor
in the slot the reference model says reads it."""
import pytest

from paper_1812_07816_b200._native import OP
from paper_1812_07816_b200.graph import tensor_bytes
from paper_1812_07816_b200.rewrite import RewriteConfig
from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer

from mock_engine import INV, dry_run

CONFIGS = [
    dict(dims=(32, 32, 32), base_filters=8, depth=3, dtype="f32", preset="paper-c1"),
    dict(dims=(32, 32, 32), base_filters=16, depth=3, dtype="bf16", preset="paper-c4"),
    dict(dims=(16, 16, 16), base_filters=16, depth=3, dtype="bf16", preset="paper-c1",
         batch=2),
    dict(dims=(192, 192, 192), base_filters=64, depth=5, dtype="bf16", preset="paper-c4"),
    dict(dims=(192, 192, 192), base_filters=64, depth=5, dtype="bf16", preset=None),
    dict(dims=(32, 32, 32), base_filters=16, depth=3, dtype="bf16", preset=None,
         rewrite=RewriteConfig(mode="recompute", ckpt_policy="speed")),
    dict(dims=(32, 32, 32), base_filters=8, depth=3, dtype="f32", preset=None,
         rewrite=RewriteConfig(mode="recompute", ckpt_policy="sqrt_n")),
    dict(dims=(192, 192, 192), base_filters=64, depth=5, dtype="bf16", preset=None,
         rewrite=RewriteConfig(mode="recompute", ckpt_policy="speed")),
    dict(dims=(192, 192, 192), base_filters=64, depth=5, dtype="bf16", preset=None,
         rewrite=RewriteConfig(mode="recompute", ckpt_policy="sqrt_n")),
    # recompute, then swap 4 of the kept checkpoints (rewrite.apply_rewrites)
    dict(dims=(192, 192, 192), base_filters=64, depth=5, dtype="bf16", preset=None,
         rewrite=(RewriteConfig(mode="recompute", ckpt_policy="speed"),
                  RewriteConfig(mode="swap", n_tensors=4, lb=40))),
]


def _cfg_id(c):
    rw = c.get("rewrite")
    if isinstance(rw, tuple):
        plan = f"rc-{rw[0].ckpt_policy}+swap{rw[1].n_tensors}"
    else:
        plan = f"rc-{rw.ckpt_policy}" if rw is not None else c["preset"]
    return f"{c['dims'][0]}-b{c['base_filters']}-{c['dtype']}-{plan}"


@pytest.fixture(scope="module", params=CONFIGS,
                ids=_cfg_id)
def trainer(request):
    return UNetTrainer(TrainConfig(**request.param), device_engine=False)


def test_residency_sound_and_plan_bytes(trainer):
    peak, d2h, h2d = dry_run(trainer.program)
    # the plan's bytes, less the swaps of BN outputs no kernel reads (elided, see
    # UNetTrainer._drop_dead_norm_outputs)
    elided = set(trainer.elided_swaps)
    assert elided <= set(trainer.plan.swapped)
    planned = sum(tensor_bytes(trainer.rw.graph.tensor(t)) for t in trainer.plan.swapped
                  if t not in elided)
    assert d2h == planned == h2d
    assert peak <= trainer.program.arena_need()


def test_prefetched_tensor_read_in_its_modelled_slot(trainer):
    pr = trainer.program
    defs = pr.by_tid()
    slot = None
    reads_in_slot: dict[int, set] = {}
    for code, tids, ia, fa in pr.ops:
        name = INV[code]
        if name == "SLOT_BEGIN":
            slot = ia[0]
        elif name == "SLOT_END":
            slot = None
        elif slot is not None and name not in ("SWAP_OUT", "FREE", "SWAP_RELEASE"):
            for t in tids:
                if t >= 0:
                    reads_in_slot.setdefault(slot, set()).add(defs[t].name)
    for t, (out_id, in_id, trigger) in trainer.plan.swapped.items():
        if t in trainer.elided_swaps:
            continue
        readers = trainer.rw.graph.consumers(t + "@in")
        # one reader (the grad slot) -- or, for a swapped recompute checkpoint, also the
        # clones recomputed from it
        assert len(readers) == 1 or trainer.plan.clone_map
        for reader in readers:
            pos = trainer.rw.position(reader)
            assert t + "@in" in reads_in_slot.get(pos, set()), (t, reader)
            # the prefetch is issued after the trigger slot, before the reader
            assert trainer.rw.position(trigger) < pos


def test_tensor_core_coverage_at_192(trainer):
    if trainer.cfg.dims[0] != 192 or trainer.plan.clone_map:
        pytest.skip("only meaningful at the production shape")
    algos = trainer.kernel_algo
    direct = sorted(k for k, v in algos.items() if v == "direct")
    # every conv/convT pass runs on tcgen05 at base 64, except (for now) the weight
    # gradient of the 4-channel input layer, whose 16-channel MN-major operand needs
    # the SWIZZLE_32B MN-major path (being validated by csrc/selftest_umma.cu T7).
    assert direct in ([], ["analysis/l0/conv1.wgrad"]), direct
    counts = {}
    for code, *_ in trainer.program.ops:
        counts[INV[code]] = counts.get(INV[code], 0) + 1
    assert counts["CONV_FWD"] == 20 and counts["CONVT_FWD"] == 4
    assert counts["CONV_WGRAD"] == 20 and counts["CONVT_WGRAD"] == 4
    assert counts["CONV_DGRAD"] == 19 and counts["CONVT_DGRAD"] == 4
    assert OP["US_OP_ADAM"] in {c for c, *_ in trainer.program.ops}


def test_no_cuda_core_conv_in_production_programs(trainer):
    """Every forward conv of a bf16 base-64 program -- recompute clones included -- runs on
    a tensor-core kernel (a stem clone once fell back to the CUDA-core direct conv)."""
    from paper_1812_07816_b200._native import ALGO_DIRECT
    if trainer.cfg.dims[0] != 192 or trainer.cfg.dtype != "bf16":
        pytest.skip("only meaningful at the production shape")
    fwd = [(op[0], op[2]) for op in trainer.program.ops
           if INV[op[0]] in ("CONV_FWD", "CONVT_FWD")]
    assert len(fwd) >= 24
    assert all(ia[7] != ALGO_DIRECT for _, ia in fwd), [ia for _, ia in fwd
                                                          if ia[7] == ALGO_DIRECT]


def test_recompute_clones_lowered_and_read_by_their_grad_slot(trainer):
    """Recompute plans (reference insert_recompute, rewrite.py:237-353): each clone slot
    writes exactly its clone tensor, grad slots read the clone instead of the forward
    tensor, and the program peak stays below the no-swap program's."""
    if trainer.plan.mode != "recompute":
        pytest.skip("recompute plans only")
    pr = trainer.program
    defs = pr.by_tid()
    rw = trainer.rw
    slot, writes, reads = None, {}, {}
    for code, tids, ia, fa in pr.ops:
        name = INV[code]
        if name == "SLOT_BEGIN":
            slot = ia[0]
        elif name == "SLOT_END":
            slot = None
        elif slot is not None and name not in ("FREE", "SWAP_RELEASE"):
            for t in tids:
                if t >= 0:
                    reads.setdefault(slot, set()).add(defs[t].name)
            if name in ("CONV_FWD", "NORM_ACT", "RELU_FWD", "POOL_FWD", "CONVT_FWD", "CONCAT"):
                writes.setdefault(slot, []).append(name)
    assert trainer.plan.clone_map
    for cid, orig in trainer.plan.clone_map.items():
        pos = rw.position(cid)
        out = rw.graph.node(cid).outputs[0]
        if out.split("@")[0] in trainer.dual_cat:
            # a dual-source concat clone is never written: its readers take its inputs
            assert not writes.get(pos), (cid, writes.get(pos))
            for reader in rw.graph.consumers(out):
                assert set(rw.graph.node(cid).inputs) <= reads[rw.position(reader)]
            continue
        assert len(writes.get(pos, ())) == 1, (cid, writes.get(pos))
        assert out in reads[pos]
        for reader in rw.graph.consumers(out):
            rnode = rw.graph.node(reader)
            if rnode.outputs and rnode.outputs[0].split("@")[0] in trainer.dual_cat:
                continue   # read by the weight gradient in place of the skipped concat clone
            assert out in reads[rw.position(reader)], (out, reader)
    peak, d2h, h2d = dry_run(pr)
    assert d2h == h2d == 0
    full = UNetTrainer(TrainConfig(dims=trainer.cfg.dims, base_filters=trainer.cfg.base_filters,
                                   depth=trainer.cfg.depth, dtype=trainer.cfg.dtype,
                                   preset=None), device_engine=False)
    assert peak < dry_run(full.program)[0]


def test_augmentation_ops_and_valid_permutations():
    """Flip / permute augmentation runs in the input conversion on the GPU:
    the loss reads the augmented labels, and only shape-preserving permutations exist."""
    cube = UNetTrainer(TrainConfig(dims=(32, 32, 32), base_filters=8, depth=3, dtype="f32",
                                   preset="paper-c1", augment=True), device_engine=False)
    assert cube.aug_perms == [0, 1, 2, 3, 4, 5]
    brats = UNetTrainer(TrainConfig(dims=(160, 240, 240), base_filters=8, depth=5, dtype="bf16",
                                    preset=None, augment=True), device_engine=False)
    assert brats.aug_perms == [0, 1]        # identity and the H <-> W swap
    pr = cube.program
    names = {d.tid: d.name for d in pr.tensors.values()}
    codes = [INV[c] for c, *_ in pr.ops]
    assert "LABELS_AUG" in codes
    for code, tids, ia, fa in pr.ops:
        if INV[code] in ("LOSS_FWD", "LOSS_BWD"):
            assert names[tids[1]] == "<labels.aug>"
        if INV[code] in ("INPUT_NCDHW", "LABELS_AUG"):
            assert len(fa) == 2
    peak, d2h, h2d = dry_run(pr)
    assert d2h == h2d > 0


def test_dead_norm_outputs_are_elided(trainer):
    """A BN output no kernel reads and no plan swaps is neither written nor allocated (the
    default "unswapped" mode: a planned swap is always executed); no op references it."""
    pr = trainer.program
    defs = pr.by_tid()
    dead = set(trainer.dead_norm_outputs)
    for code, tids, _, _ in pr.ops:
        for t in tids:
            assert t not in dead, f"dead {defs[t].name} still referenced by {INV[code]}"
    readers = {}
    for code, tids, _, _ in pr.ops:
        for t in tids:
            if t >= 0:
                readers.setdefault(t, set()).add(INV[code])
    swap_in = {tids[0]: tids[1] for code, tids, _, _ in pr.ops if INV[code] == "SWAP_IN"}
    book = {"NORM_ACT", "TOUCH", "FREE", "SWAP_OUT", "SWAP_IN", "SWAP_RELEASE"}
    for code, tids, _, _ in pr.ops:
        if INV[code] == "NORM_ACT" and tids[3] >= 0 and tids[4] >= 0:
            # kept: read by a kernel (unfused ReLU backward, recompute clone), directly
            # or through its prefetched copy
            t = tids[3]
            assert ((readers[t] - book) or (readers.get(swap_in.get(t), set()) - book)
                    or defs[t].name in trainer.plan.swapped)
    names = {defs[t].name for t in dead}
    assert not trainer.elided_swaps and not (names & set(trainer.plan.swapped))
    if trainer.plan.mode != "recompute" and trainer.cfg.dims[0] == 192:
        assert dead and all(tids[3] < 0 or defs[tids[3]].name in trainer.plan.swapped
                            for code, tids, _, _ in pr.ops
                            if INV[code] == "NORM_ACT" and tids[4] >= 0)


@pytest.mark.parametrize("preset", ["paper-c4", "paper-c1"])
def test_elide_all_skips_planned_swaps_of_dead_norm_outputs(preset):
    """elide_dead_norm="all" (the bench's elided variant) also skips the planned swaps of
    dead BN outputs and lists them; the default executes every planned swap."""
    cfg = dict(dims=(32, 32, 32), base_filters=16, depth=3, dtype="bf16", preset=preset)
    a = UNetTrainer(TrainConfig(elide_dead_norm="all", **cfg), device_engine=False)
    b = UNetTrainer(TrainConfig(**cfg), device_engine=False)
    norms = {t for t in a.plan.swapped if "/norm" in t}
    assert a.elided_swaps and set(a.elided_swaps) <= norms and not b.elided_swaps
    assert dry_run(b.program)[1] == sum(b.program.tensors[t].nbytes for t in b.plan.swapped)
    assert dry_run(a.program)[1] < dry_run(b.program)[1]
