"""Multi-GPU host logic on CPU (gloo, world size 2): communicator bootstrap, the
all-reduce placement in the lowered program, max-over-ranks timing, and the
gradient-mean semantics the device ALLREDUCE op implements."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1812_07816_b200._native import OP
from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class FakeEngine:
    def __init__(self):
        self.calls = []

    def dp_init(self, uid, world, rank):
        self.calls.append((uid, world, rank))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1812_07816_b200 import _native
        import bench
        cfg = TrainConfig(dims=(16, 16, 16), base_filters=16, depth=3, dtype="bf16",
                          preset="paper-c4", world=world)
        tr = UNetTrainer(cfg, device_engine=False)
        tr.engine = FakeEngine()
        _native.Engine.nccl_unique_id = staticmethod(lambda: b"U" * 127 + bytes([7]))
        tr.init_data_parallel(rank, world)
        uid, w, r = tr.engine.calls[0]
        # every rank receives rank 0's id and its own rank
        ok_boot = uid == b"U" * 127 + bytes([7]) and w == world and r == rank
        # max over ranks of the timed region
        t = bench.allmax(0.5 + rank, world)
        # the all-reduce mean: what the ALLREDUCE op computes on the flat gradient buffer
        import torch
        g = torch.full((8,), float(rank + 1))
        dist.all_reduce(g)
        g *= 1.0 / world
        q.put((rank, ok_boot, t, g.tolist()))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_two_rank_bootstrap_and_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_boot, t, g in res:
        assert ok_boot
        assert t == 1.5
        assert g == [1.5] * 8


@pytest.mark.parametrize("world", [1, 2, 8])
def test_allreduce_op_placement(world):
    cfg = TrainConfig(dims=(16, 16, 16), base_filters=16, depth=3, dtype="bf16",
                      preset="paper-c1", world=world)
    tr = UNetTrainer(cfg, device_engine=False)
    ops = tr.program.ops
    codes = [c for c, *_ in ops]
    adam = codes.index(OP["US_OP_ADAM"])
    ar = [k for k, c in enumerate(codes) if c == OP["US_OP_ALLREDUCE"]]
    if world == 1:
        assert not ar
        assert ops[adam][2][3] == 1    # the optimizer still overlaps the backward
        return
    assert len(ar) == 1 and ar[0] < adam
    # after every gradient producer (all wgrad ops come before it)
    last_wgrad = max(k for k, c in enumerate(codes)
                     if c in (OP["US_OP_CONV_WGRAD"], OP["US_OP_CONVT_WGRAD"]))
    assert last_wgrad < ar[0]
    _, tids, iargs, fargs = ops[ar[0]]
    # a model this small is one bucket: the whole flat buffer, on the comm stream
    assert tids == (tr.t_G,) and iargs == (0, tr.layout.total, 1)
    assert np.isclose(fargs[0], 1.0 / world)


@pytest.mark.parametrize("dims,base,depth", [((192, 192, 192), 64, 5), ((32, 32, 32), 16, 3)])
def test_gradient_buckets_cover_params_and_follow_their_wgrads(dims, base, depth):
    """Bucketed all-reduce: contiguous buckets tile the flat gradient buffer
    exactly once; each is issued on the comm stream right after the op that writes its
    last gradient, and all of them before Adam."""
    cfg = TrainConfig(dims=dims, base_filters=base, depth=depth, dtype="bf16",
                      preset="paper-c4", world=2, dp_bucket_mb=32.0)
    tr = UNetTrainer(cfg, device_engine=False)
    ops = tr.program.ops
    ar = [(k, ia) for k, (code, _, ia, _) in enumerate(ops) if code == OP["US_OP_ALLREDUCE"]]
    opt_slot = len(tr.rw.serial_order)
    adam = next(k for k, (code, _, ia, _) in enumerate(ops)
                if code == OP["US_OP_SLOT_BEGIN"] and ia[0] == opt_slot)
    # one Adam update per bucket, right behind its all-reduce, covering the same range
    adams = [(k, ia) for k, (code, _, ia, _) in enumerate(ops) if code == OP["US_OP_ADAM"]]
    assert sorted((ia[2], ia[0]) for _, ia in adams) == sorted((ia[0], ia[1]) for _, ia in ar)
    assert all(ops[k + 1][0] == OP["US_OP_ADAM"] and ops[k + 1][2][2] == ia[0] for k, ia in ar)
    spans = sorted((ia[0], ia[0] + ia[1]) for _, ia in ar)
    assert spans[0][0] == 0 and spans[-1][1] == tr.layout.total
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert all(ia[2] == 1 for _, ia in ar) and all(k < adam for k, _ in ar)
    if dims[0] == 192:
        assert len(ar) >= 8           # 640 MB of fp32 gradients, >= 32 MB buckets
    # each bucket follows the last op writing a gradient inside it
    writers = {OP["US_OP_CONV_WGRAD"]: (6,), OP["US_OP_CONVT_WGRAD"]: (6,),
               OP["US_OP_BN_BWD"]: (4, 5), OP["US_OP_LOSS_BWD"]: (6, 7)}
    for k, ia in ar:
        lo, hi = ia[0], ia[0] + ia[1]
        last = max(j for j, (code, _, ja, _) in enumerate(ops)
                   if code in writers and any(lo <= ja[q] < hi for q in writers[code]))
        assert last < k
        assert all(ops[j][0] in (OP["US_OP_ALLREDUCE"], OP["US_OP_ADAM"], OP["US_OP_FREE"])
                   for j in range(last + 1, k))


def _dp_program_worker(rank, world, port, q):
    """Lower the real data-parallel program (192^3, depth 5, base 64, paper-c4) on this rank
    and run its ALLREDUCE ops -- in program order, on the flat gradient buffer -- as gloo
    collectives over per-rank gradients."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import hashlib
        import torch
        cfg = TrainConfig(dims=(192, 192, 192), base_filters=64, depth=5, dtype="bf16",
                          preset="paper-c4", world=world, device=rank)
        tr = UNetTrainer(cfg, device_engine=False)
        ar = [(k, ia, fa) for k, (code, _, ia, fa) in enumerate(tr.program.ops)
              if code == OP["US_OP_ALLREDUCE"]]
        digest = hashlib.sha256(repr([(c, t, i) for c, t, i, _ in tr.program.ops])
                                .encode()).hexdigest()
        # the collectives every rank issues, in order: must be identical or NCCL deadlocks
        sched = [(k, tuple(ia), tuple(fa)) for k, ia, fa in ar]
        got = [None] * world
        dist.all_gather_object(got, (sched, digest))
        same = all(g == got[0] for g in got)
        # gradient mean through the program's buckets
        total = tr.layout.total
        g = torch.arange(total, dtype=torch.float32) % 97 + 1000.0 * (rank + 1)
        for _, ia, fa in ar:
            off, count = ia[0], ia[1]
            seg = g[off:off + count]
            dist.all_reduce(seg)
            seg.mul_(fa[0])
            g[off:off + count] = seg
        expect = torch.arange(total, dtype=torch.float32) % 97 + 1000.0 * (world + 1) / 2
        ok_mean = bool(torch.allclose(g, expect))
        q.put((rank, same, len(ar), ok_mean, total))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_two_rank_dp_program_identical_buckets_and_mean():
    """World 2 on gloo: both ranks lower the same DP program (same ops, same bucket tiling
    and ALLREDUCE placement, so the NCCL collectives match), and executing its buckets
    averages the per-rank gradients over the whole flat buffer."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_program_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, n_ar, ok_mean, total in res:
        assert same and ok_mean
        assert n_ar >= 8 and total > 160_000_000


def test_bench_refuses_more_gpus_than_visible():
    """bench.py --gpus N outside torchrun re-launches itself with N ranks, and refuses when
    fewer GPUs are visible (here: none)."""
    import subprocess
    import sys
    import bench
    if bench.visible_gpus() >= 4:
        pytest.skip("this host has 4 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--steps", "1"], cwd=root,
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 2
    assert "only" in r.stderr and "visible" in r.stderr
