#!/usr/bin/env python
"""Benchmark: full-volume 3D U-Net training step with data swapping on B200.

Metric (BASELINE.json): 192^3 3D U-Net train voxels/s, plus exposed swap
overhead as % of the step.  Default workload (configs[2]): 4x192^3, batch 1 per
GPU, depth 5 / base 64, swap plan = the paper-default preset (paper-c4)
EXECUTED BYTE FOR BYTE (every planned swap-out and prefetch moves its bytes),
bf16 tensor-core kernels, Adam.  One step = forward + soft-Dice loss + backward
+ (all-reduce) + Adam over one synthetic BraTS-shaped volume per GPU.

    python bench.py [--gpus N --steps K --warmup W] [--config NAME] [plan flags]
    python bench.py --impl reference ...        # the reference arm (CPU)

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one process per GPU); it fails loudly when fewer than N GPUs are visible.
Plan flags mirror the reference CLI (cli.py:322-408): --preset, --mode,
--n-tensors, --lb, --excl-scopes, --incl-scopes, --ckpt-policy.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (dims, batch, plan, description)
    #   plan: preset name | None | "tuned:<GiB>:<swap|all>" | "recompute:<policy>"
    "f192-c4": ((192, 192, 192), 1, "paper-c4",
                "4x192^3 b1 paper-c4 (paper-default swap, executed byte for byte)"),
    "f192-noswap": ((192, 192, 192), 1, None, "4x192^3 b1 no swap"),
    "f192-c1": ((192, 192, 192), 1, "paper-c1", "4x192^3 b1 paper-c1 (swap all)"),
    "p128-b2": ((128, 128, 128), 2, None, "4x128^3 b2 patch baseline, no swap"),
    # configs[3]: plan tuned by the engine model under an HBM budget the unswapped step does
    # not fit (engine no-swap peak at 192^3: 11.15 GiB) -- only swap plans compete
    "f192-tuned": ((192, 192, 192), 1, "tuned:11:swap", "4x192^3 b1, swap plan tuned for an "
                   "11 GiB arena (the unswapped step needs 11.15 GiB)"),
    "f192-tuned-10": ((192, 192, 192), 1, "tuned:10:swap", "4x192^3 b1, swap plan tuned for a "
                      "10 GiB arena"),
    "f192-tuned-8": ((192, 192, 192), 1, "tuned:8:all", "4x192^3 b1, plan (swap, recompute or "
                     "both) tuned for an 8 GiB arena"),
    # the paper's section-5 alternative: recompute instead of swap
    "f192-rc-speed": ((192, 192, 192), 1, "recompute:speed", "4x192^3 b1 recompute, "
                      "speed policy (keep conv outputs)"),
    "f192-rc-sqrt": ((192, 192, 192), 1, "recompute:sqrt_n", "4x192^3 b1 recompute, "
                     "sqrt(n) checkpoints"),
    # configs[4]: native BraTS extent (155 slices padded to 160), batch raised until the
    # step no longer fits a 180 GB B200 without swapping (b = 12: the unswapped step needs
    # ~174 GiB of step tensors)
    "n240-b12-tuned": ((160, 240, 240), 12, "tuned:171:swap", "4x240x240x160 b12, swap plan "
                       "tuned for a 171 GiB arena (the unswapped step needs 174.2 GiB)"),
    "n240-b8-tuned": ((160, 240, 240), 8, "tuned:120:swap", "4x240x240x160 b8, swap plan tuned "
                      "for a 120 GiB arena"),
}
CPU_SAMPLE_DIMS = (48, 48, 48)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------- launch

def self_launch(args, argv) -> None:
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run, one rank per
    GPU.  Fails loudly when fewer GPUs are visible than asked for."""
    n_vis = visible_gpus()
    if n_vis < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {n_vis} GPU(s) are visible",
              file=sys.stderr)
        sys.exit(2)
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + argv
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr,
          flush=True)
    os.execv(sys.executable, cmd)


def visible_gpus() -> int:
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=30)
        n = sum(1 for line in out.stdout.splitlines() if line.startswith("GPU "))
    except (OSError, subprocess.TimeoutExpired):
        n = 0
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis is not None:
        n = min(n, len([v for v in vis.split(",") if v.strip()]))
    return n


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # host-side control plane (barrier, max-over-ranks, the NCCL unique id); the
        # gradient all-reduce runs inside the engine on its own NCCL communicator
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


def allmax(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------- plans

def rewrite_from_args(args, plan):
    """RewriteConfig from the reference-CLI flags (cli.py:66-78), else from the config."""
    from paper_1812_07816_b200.rewrite import RewriteConfig, resolve_preset
    if args.preset:
        return resolve_preset(args.preset), args.preset
    if args.mode:
        split = lambda s: tuple(x for x in (s or "").split(",") if x)   # noqa: E731
        cfg = RewriteConfig(mode=args.mode, n_tensors=args.n_tensors, lb=args.lb,
                            excl_scopes=split(args.excl_scopes),
                            incl_scopes=split(args.incl_scopes), ckpt_policy=args.ckpt_policy)
        return cfg, (f"{args.mode} n_tensors={args.n_tensors} lb={args.lb} "
                     f"excl={args.excl_scopes or '-'} incl={args.incl_scopes or '-'}")
    if plan is None:
        return RewriteConfig(mode="none"), "none"
    if plan.startswith("recompute:"):
        return RewriteConfig(mode="recompute", ckpt_policy=plan.split(":")[1]), plan
    return resolve_preset(plan), plan


def measure_link(local: int) -> dict:
    """Pinned host <-> HBM copy bandwidth, each direction alone and both at once (the
    swap engine's binding resource), 1 GiB per copy, best of 3."""
    import torch
    dev = torch.device("cuda", local)
    n = 1 << 30
    h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn):
        best = float("inf")
        for _ in range(3):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize(dev)
            best = min(best, time.perf_counter() - t0)
        return best

    def d2h():
        with torch.cuda.stream(s1):
            h1.copy_(d1, non_blocking=True)

    def h2d():
        with torch.cuda.stream(s2):
            d2.copy_(h2, non_blocking=True)

    def both():
        d2h()
        h2d()

    out = {"d2h_gbs": n / timed(d2h) / 1e9, "h2d_gbs": n / timed(h2d) / 1e9}
    tb = timed(both)
    out["duplex_gbs_per_direction"] = n / tb / 1e9
    del h1, h2, d1, d2
    torch.cuda.empty_cache()
    return out


def probe_slot_times(dims, batch, local, elide="unswapped"):
    """Per-slot compute seconds of the no-swap step (timeline mode), the tuner's
    calibration.  When the batch cannot run unswapped on one GPU, probe batch 1 and
    scale (every op is linear in the batch)."""
    from paper_1812_07816_b200.engine_model import slot_times_from_timeline
    from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer
    pb = batch
    full = UNetTrainer(TrainConfig(dims=dims, batch=batch, preset=None, dtype="bf16",
                                   elide_dead_norm=elide), device_engine=False)
    if full.program.order_peak() > 150 * (1 << 30):
        pb = 1
    probe = UNetTrainer(TrainConfig(dims=dims, batch=pb, preset=None, dtype="bf16",
                                    device=local, elide_dead_norm=elide))
    x, y = probe.synthetic_batch(seed=0)
    probe.load_batch(x, y)
    for _ in range(3):
        probe.step()
    rep = probe.timeline()
    probe.close()
    return slot_times_from_timeline(rep, scale=batch / pb), pb


def tune(dims, batch, budget_gib, local, elide, link, modes="swap"):
    """Engine-aware tuning (tune.tune_for_budget) under an arena of budget_gib.

    modes "swap": the paper's regime -- only swap plans compete (forced swapping); the
    best plan of the wider search (recompute and recompute+swap mixes) is reported beside
    it as a prediction.  modes "all": every plan competes."""
    from paper_1812_07816_b200.tune import tune_for_budget
    from paper_1812_07816_b200.unet import TrainConfig
    slots, pb = probe_slot_times(dims, batch, local, elide)
    base = TrainConfig(dims=dims, batch=batch, preset=None, dtype="bf16",
                       elide_dead_norm=elide)
    bw_d = link["duplex_gbs_per_direction"] * 1e9
    budget = int(budget_gib * (1 << 30))
    t0 = time.perf_counter()
    ranked = tune_for_budget(base, slots, bw_d, bw_d, budget, modes=modes)
    info = {"budget_gib": budget_gib, "tune_modes": modes, "probe_batch": pb,
            "tuning_s": time.perf_counter() - t0,
            "link_gbs_used": bw_d / 1e9, "feasible_candidates": len(ranked),
            "no_swap_compute_ms": 1e3 * sum(slots.values())}
    # does the budget bind?  Lay out the unswapped program in it (host only, no device)
    import dataclasses
    from paper_1812_07816_b200.unet import UNetTrainer
    try:
        UNetTrainer(dataclasses.replace(base, arena_bytes=budget, slot_seconds=slots,
                                        link_gbs=bw_d / 1e9), device_engine=False)
        info["unswapped_step_at_budget"] = "fits"
    except Exception as exc:   # noqa: BLE001 -- InfeasibleError / DeadlockError
        info["unswapped_step_at_budget"] = f"{type(exc).__name__}: {exc}"[:300]
    if modes == "swap":
        wider = tune_for_budget(base, slots, bw_d, bw_d, budget, modes="all")
        info["best_any_plan_predicted"] = wider[0].summary() if wider else None
    return ranked, info


# ---------------------------------------------------------------------------- CPU side

def cpu_reference(dims, batch, steps: int = 2, warmup: int = 0):
    """The real-op CPU restatement (oracle/unet_fp64.py, torch fp32, all host threads) on
    a bounded crop of the same U-Net.  Builds its parameters and input without the CUDA
    library.  Returns (voxels/s, threads, sample description, s/step)."""
    import torch
    from oracle.unet_fp64 import cpu_train_step_seconds, init_params, synthetic_batch
    from paper_1812_07816_b200.models import gen_unet3d
    from paper_1812_07816_b200.unet import TrainConfig
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg = TrainConfig(dims=CPU_SAMPLE_DIMS, batch=1, preset=None, dtype="f32")
    params = init_params(gen_unet3d(cfg.unet_params()), cfg.seed, cfg.n_classes)
    x, y = synthetic_batch(cfg.dims, 1, cfg.in_channels, cfg.n_classes, seed=0)
    sec, used = cpu_train_step_seconds(cfg, params, x, y, steps=steps, warmup=warmup)
    vox = CPU_SAMPLE_DIMS[0] * CPU_SAMPLE_DIMS[1] * CPU_SAMPLE_DIMS[2]
    sample = (f"4x{CPU_SAMPLE_DIMS[0]}^3 crop (batch 1) of the {dims[0]}x{dims[1]}x{dims[2]} "
              f"b{batch} workload: same depth-5/base-64 U-Net, torch-CPU fp32 "
              f"fwd+Dice+bwd+Adam, best of {steps} steps ({sec:.2f} s/step)")
    return vox / sec, used, sample, sec


def reference_cpu_path() -> dict:
    """The reference's own CPU path: planner
    (gen_unet3d + expand_training_graph + apply_rewrite, 192^3 paper-c4), simulate +
    stall_report, and the toy run_numeric train step at the tiny config (4x32^3, depth 3,
    base 8, paper-c4, MAX_ELEMENTS raised) -- from the unmodified reference installed in
    baseline/_ref when present, else from the restatements (package planner + oracle
    toy executor)."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    kind = "port"
    if os.path.isdir(os.path.join(ref_dir, "swapsim")):
        sys.path.insert(0, ref_dir)
        import swapsim.numeric as num
        from swapsim import (UNetParams, apply_rewrite, expand_training_graph, gen_unet3d,
                             resolve_preset, simulate, stall_report)
        from swapsim.sim import SimConfig
        run_numeric = num.run_numeric
        num.MAX_ELEMENTS = 1 << 24
        kind = "reference"
        sys.path.remove(ref_dir)
    else:
        from oracle.toy_numeric import run_numeric
        from paper_1812_07816_b200 import (UNetParams, apply_rewrite, expand_training_graph,
                                           gen_unet3d, resolve_preset, simulate,
                                           stall_report)
        from paper_1812_07816_b200.sim import SimConfig

    def best(fn, n):
        t = float("inf")
        for _ in range(n):
            t0 = time.perf_counter()
            r = fn()
            t = min(t, time.perf_counter() - t0)
        return t, r

    def plan():
        tg = expand_training_graph(gen_unet3d(UNetParams(dims=(192, 192, 192), elem_bytes=2)))
        return apply_rewrite(tg, resolve_preset("paper-c4"))

    t_plan, (rw, pl) = best(plan, 5)
    t_sim, _ = best(lambda: stall_report(simulate(rw, pl, SimConfig(d2h_bw=55e9,
                                                                     h2d_bw=55e9))), 5)
    tiny = expand_training_graph(gen_unet3d(UNetParams(dims=(32, 32, 32), in_channels=4,
                                                       base_filters=8, depth=3)))
    trw, tpl = apply_rewrite(tiny, resolve_preset("paper-c4"))
    t_toy, _ = best(lambda: run_numeric(trw, tpl, 1), 3)
    return {"kind": kind, "cores": 1, "planner_ms": 1e3 * t_plan, "simulate_ms": 1e3 * t_sim,
            "toy_run_numeric_ms_per_step": 1e3 * t_toy,
            "toy_run_numeric_voxels_per_s": 32 ** 3 / t_toy,
            "sample": "planner + simulate/stall_report at 192^3 paper-c4; run_numeric "
                      "(toy arithmetic, fp64 numpy) at 4x32^3 depth 3 base 8 paper-c4"}


def config_dict(desc, batch, world, plan_label):
    return {"workload": desc, "model": "3D U-Net depth 5 base 64 (gen_unet3d)",
            "global_batch": batch * world, "seq_len": None, "parallelism": f"dp{world}",
            "swap_plan": plan_label,
            "l2": "inputs and activations (0.1-1.8 GB per tensor) exceed the 126 MB L2"}


def run_reference(args, world, rank):
    """The reference arm: the real-op CPU restatement on all host cores, each step a
    bounded crop of the workload (the reference itself has no real-op implementation),
    plus the reference's own CPU path.  Never loads the CUDA library."""
    dims, batch, plan, desc = CONFIGS[args.config]
    if rank != 0:
        return
    _, plan_label = rewrite_from_args(args, plan if not (plan or "").startswith("tuned")
                                      else None)
    if (plan or "").startswith("tuned"):
        plan_label = "tuned"
    v, threads, sample, sec = cpu_reference(dims, batch, steps=args.steps, warmup=args.warmup)
    vox_full = dims[0] * dims[1] * dims[2] * batch
    line = {
        "impl": "reference", "metric": "192^3 3D U-Net train voxels/s", "value": v,
        "unit": "voxels/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * vox_full / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(desc, batch, args.gpus, plan_label),
        "sample": sample,
        "cpu_baseline": {"value": v, "unit": "voxels/s", "cores": threads, "kind": "port",
                         "sample": sample, "reference_cpu_path": reference_cpu_path()},
        "e2e": {"value": v, "unit": "voxels/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU side

def build_trainer(dims, batch, rewrite, args, world, rank, local, arena):
    from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer
    cfg = TrainConfig(dims=dims, batch=batch, preset=None, rewrite=rewrite, dtype="bf16",
                      world=world, device=local, seed=0, arena_bytes=arena,
                      graph=not args.no_graph, d2h_order=args.d2h_order, augment=args.augment,
                      elide_dead_norm="all" if args.elide_dead_norm else "unswapped",
                      direct_concat=not args.no_direct_concat,
                      dual_source_concat=not args.no_dual_source,
                      fuse_bn_sums={"off": False, "all": True, "dgrad": "dgrad"}[
                          args.fuse_bn_sums])
    tr = UNetTrainer(cfg)
    tr.init_data_parallel(rank, world)
    if world > 1 or cfg.dp_force_allreduce:
        n = tr.engine.stats()["dp_nranks"]
        print(f"bench.py rank {rank}: NCCL communicator nranks={n} (device {local})",
              file=sys.stderr, flush=True)
        if n != world:
            raise RuntimeError(f"NCCL communicator has {n} ranks, expected {world}")
    x, y = tr.synthetic_batch(seed=rank)
    tr.load_batch(x, y)
    tr.step()
    return tr, x, y


def timed_steps(tr, steps, warmup, world):
    """Device-timed loop (CUDA events on the compute stream), inputs resident in HBM,
    after `warmup` untimed steps (the CUDA graph is captured on the 3rd run)."""
    from paper_1812_07816_b200._native import FLAG_NO_TIMELINE
    tr.engine.set_flags(tr.engine.flags | FLAG_NO_TIMELINE)
    for _ in range(max(3, warmup)):
        tr.step()
    barrier(world)
    tr.engine.mark(0)
    for _ in range(steps):
        tr.run_async()
    tr.engine.mark(1)
    t = tr.engine.elapsed()
    tr.engine.sync()
    return allmax(t, world)


def run_ours(args, world, rank, local):
    import numpy as np
    from paper_1812_07816_b200.sim import stall_report
    dims, batch, plan, desc = CONFIGS[args.config]
    link = measure_link(local)
    tuned = None
    arena = int(args.budget_gb * (1 << 30)) if args.budget_gb else None
    if (plan or "").startswith("tuned:") and not (args.preset or args.mode):
        budget = args.budget_gb or float(plan.split(":")[1])
        modes = args.tune_modes or plan.split(":")[2]
        ranked, tuned = tune(dims, batch, budget, local,
                             "all" if args.elide_dead_norm else "unswapped", link, modes)
        if not ranked:
            raise SystemExit(f"bench.py: no plan fits a {budget} GiB arena")
        arena = int(budget * (1 << 30))
        tr = None
        tried = []
        for cand in ranked[:4]:   # same budget; a plan the allocator cannot place is skipped
            try:
                tr, x, y = build_trainer(dims, batch, cand.rewrite, args, world, rank, local,
                                         arena)
                break
            except Exception as exc:   # noqa: BLE001 -- InfeasibleError / DeadlockError
                tried.append({"label": cand.label, "error": str(exc)[:200]})
                if tr is not None:
                    tr.close()
                tr = None
        if tr is None:
            raise SystemExit(f"bench.py: no tuned plan ran in {budget} GiB: {tried}")
        tuned.update(cand.summary())
        tuned["rejected_by_allocator"] = tried
        tuned["top5"] = [c.summary() for c in ranked[:5]]
        plan_label = "tuned: " + cand.label
    else:
        rewrite, plan_label = rewrite_from_args(args, plan)
        tr, x, y = build_trainer(dims, batch, rewrite, args, world, rank, local, arena)

    # timeline steps: per-slot / per-copy timestamps for the swap statistics and the
    # exposed-swap fraction (timed events cost ~40 us each while PCIe is saturated, so the
    # measured loop runs without them)
    for _ in range(3):
        tr.step()
    st = tr.engine.stats()
    rep = tr.timeline()
    phys_peak = tr.physical_peak(rep)
    stalls = stall_report(rep)
    busy = {"d2h": 0.0, "h2d": 0.0}
    for _, ch, s0, e0 in rep.events:
        if ch in busy:
            busy[ch] += e0 - s0
    if args.trace and rank == 0:
        from paper_1812_07816_b200.sim import emit_trace
        emit_trace(rep, args.trace)

    clocks = ClockSampler(local)
    clocks.start()
    t_max = timed_steps(tr, args.steps, args.warmup, world)
    clk = clocks.stop()
    st_timed = tr.engine.stats()
    kernels_per_step = st_timed["kernels"]
    vox = dims[0] * dims[1] * dims[2] * batch
    value = world * vox * args.steps / t_max

    # end-to-end through the public API: pinned host volume + labels -> device every
    # step, the loss read back
    import torch
    xp = torch.empty(x.size, dtype=torch.float32, pin_memory=True)
    yp = torch.empty(y.size, dtype=torch.uint8, pin_memory=True)
    xp.numpy()[:] = x.reshape(-1)
    yp.numpy()[:] = y.reshape(-1)
    barrier(world)
    tr.engine.mark(0)
    losses = []
    for _ in range(args.steps):
        tr.load_batch_ptr(xp.data_ptr(), yp.data_ptr())
        tr.run_async()
        losses.append(float(tr.engine.download(tr.t_LOSS, 4, np.float32)[0]))
    tr.engine.mark(1)
    t_e2e = allmax(tr.engine.elapsed(), world)
    e2e = world * vox * args.steps / t_e2e

    # per-op kernel times (CUDA events on the compute stream, after residency waits)
    pk, pk_kind = peaks()
    optimes = tr.op_times(3)
    if args.op_dump and rank == 0:
        with open(args.op_dump, "w") as f:
            json.dump([{"op": k, "name": name, "slot": slot, "ms": 1e3 * t,
                        "iargs": list(tr.program.ops[k][2])}
                       for k, name, slot, t in optimes], f, indent=0)
    conv_nodes = {n.id: n for n in tr.graph.nodes if n.kind == "conv"}
    conv_t = sum(t for _, name, slot, t in optimes if name == "CONV_FWD" and slot in conv_nodes)
    conv_flops = sum(n.cost_units for n in conv_nodes.values()) * batch
    achieved = conv_flops / conv_t / 1e12 if conv_t > 0 else 0.0
    peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    kern = {}
    for _, name, slot, t in optimes:
        kern[name] = kern.get(name, 0.0) + t
    top = sorted(optimes, key=lambda r: -r[3])[:10]
    conv_ops = ("CONV_FWD", "CONV_DGRAD", "CONV_WGRAD", "CONVT_FWD", "CONVT_DGRAD",
                "CONVT_WGRAD")
    dom_slot = "analysis/l0/conv2"
    dom_t = sum(t for _, name, slot, t in optimes if name == "CONV_FWD" and slot == dom_slot)
    dom_flops = conv_nodes[dom_slot].cost_units * batch if dom_slot in conv_nodes else 0.0
    dom_prof = {}
    prof_path = os.path.join(ROOT, "profiles", "r02_dominant_kernel.json")
    if not os.path.exists(prof_path):
        prof_path = os.path.join(ROOT, "profiles", "r01_dominant_kernel.json")
    if os.path.exists(prof_path) and dims == (192, 192, 192) and batch == 1:
        with open(prof_path) as f:
            dom_prof = json.load(f)
    dominant = {"slot": dom_slot, "kernel": dom_prof.get("kernel", "k_halo_z2<fprop>"),
                "ms": 1e3 * dom_t,
                "achieved_tflops": dom_flops / dom_t / 1e12 if dom_t > 0 else None,
                "frac_of_sustained": (dom_flops / dom_t / 1e12 / peak) if dom_t > 0 else None,
                "frac_of_burst": (dom_flops / dom_t / 1e12 / pk.get("bf16_tflops", peak))
                if dom_t > 0 else None,
                "dram_bytes_per_launch": dom_prof.get("dram_bytes"),
                "algorithmic_min_bytes": dom_prof.get("algorithmic_min_bytes"),
                "tensor_pipe_active_pct_ncu": dom_prof.get("tensor_pipe_active_pct"),
                "profile": os.path.basename(prof_path) if dom_prof else None}
    step_flops = 3.0 * sum(n.cost_units for n in tr.graph.nodes
                           if n.kind in ("conv", "upsample")) * batch
    step_s = st["step_s"]
    planned = int(sum(tr.program.tensors[t].nbytes for t in tr.plan.swapped))
    moved = st["d2h_bytes"]
    link_busy = max(busy.values()) if busy else 0.0
    link_roof = {"bound": "pcie", "unit": "GB/s",
                 "achieved_d2h_while_busy": moved / busy["d2h"] / 1e9 if busy["d2h"] else None,
                 "achieved_h2d_while_busy": st["h2d_bytes"] / busy["h2d"] / 1e9
                 if busy["h2d"] else None,
                 "peak_measured": link,
                 "link_busy_frac_of_step": link_busy / step_s if step_s else None}
    step_meas = t_max / args.steps
    both = (moved + st["h2d_bytes"]) / step_meas / 1e9 if step_meas else 0.0
    link_roof["achieved_both_directions_gbs"] = both   # over the whole (untimed) step
    if link.get("duplex_gbs_per_direction"):
        # whole-step link utilisation against its measured capacity with both directions
        # busy (2 x the per-direction duplex rate)
        link_roof["peak"] = 2 * link["duplex_gbs_per_direction"]
        link_roof["frac"] = both / link_roof["peak"]

    tr.close()
    # the elided variant (extra key): the same plan with BatchNorm outputs no kernel reads
    # left unwritten and their planned swaps skipped
    elided = None
    if (not args.elide_dead_norm and not args.no_elided_variant and tuned is None
            and any("/norm" in t for t in tr.plan.swapped)):
        args_e = argparse.Namespace(**vars(args))
        args_e.elide_dead_norm = True
        te, _, _ = build_trainer(dims, batch, tr.rcfg, args_e, world, rank, local, arena)
        for _ in range(2):
            te.step()
        ste = te.engine.stats()
        t_e = timed_steps(te, args.steps, args.warmup, world)
        elided = {"value": world * vox * args.steps / t_e, "ms_per_step": 1e3 * t_e / args.steps,
                  "d2h_bytes_per_step": ste["d2h_bytes"],
                  "exposed_swap_pct": 100.0 * ste["stall_s"] / ste["step_s"]
                  if ste["step_s"] else None,
                  "elided_swaps": len(te.elided_swaps),
                  "note": "NOT the headline: BatchNorm outputs no kernel reads (fused NORM_ACT) "
                          "are not written and their planned swaps are skipped"}
        te.close()

    # epoch model (reference sim.epoch_time, sim.py:343-348; paper: 171 full volumes per
    # epoch, flip/permute augmentation each iteration)
    from paper_1812_07816_b200.sim import epoch_time
    step_s_meas = t_max / args.steps
    epoch = {"iterations": 171, "step_s": step_s_meas,
             "epoch_s": epoch_time(step_s_meas, 171, 0.0), "paper_epoch_s": 670.0}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:   # N = 1 only (host cores
        v, threads, sample, _ = cpu_reference(dims, batch, steps=2, warmup=1)   # are shared)
        cpu = {"value": v, "unit": "voxels/s", "cores": threads, "kind": "port",
               "sample": sample, "reference_cpu_path": reference_cpu_path()}
    if rank != 0:
        return
    line = {
        "metric": "192^3 3D U-Net train voxels/s", "value": value, "unit": "voxels/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) 4-modality "
        "volume, uniform labels, Kaiming-init weights)",
        "config": config_dict(desc, batch, world, plan_label),
        "exposed_swap_pct": 100.0 * st["stall_s"] / step_s if step_s else None,
        "exposed_swap_note": "compute-stream stalls / step, from 3 timeline steps",
        "swap": {"d2h_bytes_per_step": moved, "h2d_bytes_per_step": st["h2d_bytes"],
                 "planned_swap_bytes": planned,
                 "executed_byte_for_byte": moved == planned == st["h2d_bytes"],
                 "swapped_tensors": len(tr.plan.swapped),
                 "recompute_clones": len(tr.plan.clone_map),
                 "elided_swaps": len(tr.elided_swaps),
                 "stall_s": st["stall_s"], "stall_split_s": stalls,
                 "arena_budget_bytes": arena, "arena_peak_bytes": st["arena_peak_bytes"],
                 "physical_peak_bytes": phys_peak,
                 "host_pool_bytes": st["host_pool_bytes"],
                 "host_pool_numa_node": st["host_numa_node"],
                 "d2h_order": tr.d2h_order,
                 "d2h_busy_s": busy["d2h"], "h2d_busy_s": busy["h2d"],
                 "planner_static_peak_bytes": tr.liveness.peak_bytes},
        "step_tflops": step_flops / (t_max / args.steps) / 1e12,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None,
                     # the same against the burst peak (the PCIe-bound step leaves the GPU
                     # idle much of the time, so its convs run at near-burst clocks)
                     "frac_of_burst": achieved / pk["bf16_tflops"] if pk.get("bf16_tflops")
                     else None,
                     "traffic": dom_prof.get("dram_bytes"),
                     "traffic_note": "DRAM bytes per launch of the dominant conv fprop kernel "
                                     "(ncu --set full)",
                     "dominant_kernel": dominant,
                     "kernel": "conv fprop (tcgen05), 20 conv forward ops, per-op CUDA events",
                     "kernel_ms_per_step": 1e3 * conv_t,
                     "peak_kind": f"{pk_kind} bf16_tflops_sustained"},
        "link_roofline": link_roof,
        "op_ms_per_step": {k: round(1e3 * v, 3) for k, v in sorted(kern.items(),
                                                                   key=lambda kv: -kv[1])},
        "conv_ms_per_step": round(1e3 * sum(kern.get(k, 0.0) for k in conv_ops), 3),
        "top_ops": [[name, slot, round(1e3 * t, 3)] for _, name, slot, t in top],
        "cpu_baseline": cpu,
        "tuned_plan": tuned,
        "elided_variant": elided,
        "e2e": {"value": e2e, "unit": "voxels/s",
                "h2d_bytes_per_step": int(x.nbytes + y.nbytes), "d2h_bytes_per_step": 4},
        "epoch_model": epoch,
        "augment": bool(args.augment),
        "gpu_launches": kernels_per_step * args.steps,
        "timeline_step_ms": 1e3 * st["step_s"],
        "clocks": clk,
        "loss_last": losses[-1] if losses else None,
    }
    if tuned is not None:
        tuned["measured_ms"] = 1e3 * step_s
        tuned["measured_exposed_pct"] = line["exposed_swap_pct"]
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="f192-c4")
    # plan flags (reference cli.py:322-408); override the config's plan
    ap.add_argument("--preset", default=None, help="paper-c1..c4")
    ap.add_argument("--mode", choices=["swap", "recompute", "none"], default=None)
    ap.add_argument("--n-tensors", type=int, default=-1)
    ap.add_argument("--lb", type=int, default=1)
    ap.add_argument("--excl-scopes", default="")
    ap.add_argument("--incl-scopes", default="")
    ap.add_argument("--ckpt-policy", choices=["speed", "sqrt_n"], default="speed")
    ap.add_argument("--tune-modes", choices=["swap", "all"], default=None,
                    help="tuned configs (default: the config's): 'swap' = only swap plans "
                         "compete (the paper's forced-swap regime; the best recompute/mixed "
                         "plan is reported as a prediction), 'all' = swap, recompute and "
                         "mixed plans compete")
    ap.add_argument("--budget-gb", type=float, default=None,
                    help="arena (HBM budget for step tensors, GiB); a plan that does not fit "
                         "fails with InfeasibleError / DeadlockError -- never grown")
    ap.add_argument("--elide-dead-norm", action="store_true",
                    help="do not write BatchNorm outputs no kernel reads and skip their "
                         "planned swaps (the default executes the plan byte for byte)")
    ap.add_argument("--no-elided-variant", action="store_true",
                    help="skip the extra measurement of the elided variant")
    ap.add_argument("--d2h-order", choices=["need", "fifo"], default="need")
    ap.add_argument("--augment", action="store_true")
    ap.add_argument("--fuse-bn-sums", choices=["off", "all", "dgrad"], default="off")
    ap.add_argument("--no-direct-concat", action="store_true")
    ap.add_argument("--no-dual-source", action="store_true",
                    help="materialise the synthesis concats instead of two-source convs")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trace", default=None)
    ap.add_argument("--op-dump", default=None)
    argv = sys.argv[1:]
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        self_launch(args, argv)
    world, rank, local = dist_env()
    if args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
