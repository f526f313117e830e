"""Generate the golden fixtures the parity tests compare against.

Run in the build container (the reference is not present on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the UNMODIFIED reference package from /root/reference/pkg/src
(read-only) and records, for every configuration the tests use:
  * plan JSON bytes (RewritePlan.to_json) and their sha256,
  * canonical training-graph / rewritten-graph JSON sha256,
  * select_swap_tensors order, static_peak_estimate,
  * simulate() reports + stall_report,
  * run_numeric() (toy executor) loss and input gradients.
Outputs: tests/golden/planner.json, tests/golden/sim.json,
tests/golden/numeric_*.npz.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import swapsim  # noqa: E402
from swapsim import numeric as ref_numeric  # noqa: E402
from swapsim.graph import dumps_canonical, graph_to_obj  # noqa: E402
from swapsim.models import UNetParams, gen_chain, gen_unet3d  # noqa: E402
from swapsim.rewrite import (PRESETS, RewriteConfig, apply_rewrite,  # noqa: E402
                             resolve_preset, select_swap_tensors)
from swapsim.sim import SimConfig, simulate, stall_report  # noqa: E402
from swapsim.training import (cross_phase_tensors, expand_training_graph,  # noqa: E402
                              static_peak_estimate, training_to_obj)

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


# name -> (generator kwargs) ; kept in sync with tests/golden_configs.py
UNET_CONFIGS = {
    "toy8": dict(dims=(8, 8, 8), in_channels=1, base_filters=1, depth=2, convs_per_level=1),
    "u16": dict(dims=(16, 16, 16), in_channels=1, base_filters=2, depth=3),
    "tiny": dict(dims=(32, 32, 32), in_channels=4, base_filters=8, depth=3),
    "tiny_bf16": dict(dims=(32, 32, 32), in_channels=4, base_filters=8, depth=3, elem_bytes=2),
    "p128": dict(dims=(128, 128, 128), elem_bytes=4),
    "f192": dict(dims=(192, 192, 192)),
    "f192_bf16": dict(dims=(192, 192, 192), elem_bytes=2),
    "n240": dict(dims=(240, 240, 160), elem_bytes=2),
    "f208": dict(dims=(208, 208, 208)),
}
CHAIN_CONFIGS = {
    "chain5": dict(n=5),
    "chain9_mixed": dict(n=9, bytes_per_tensor=640, kinds=("conv", "activation", "norm")),
    "chain50": dict(n=50, bytes_per_tensor=64, kinds=("conv", "activation", "norm")),
}


def build(name):
    if name in UNET_CONFIGS:
        return gen_unet3d(UNetParams(**UNET_CONFIGS[name]))
    kw = dict(CHAIN_CONFIGS[name])
    n = kw.pop("n")
    return gen_chain(n, **kw)


def random_cfgs(tg, seed, count):
    rng = random.Random(seed)
    scopes = ["analysis/*", "synthesis/*", "bottleneck/*", "*/l0/*", "*/l1/*", "chain/op1",
              "analysis/l0/*", "*norm*", "*act*"]
    n_cand = len(cross_phase_tensors(tg))
    out = []
    for _ in range(count):
        out.append(dict(
            n_tensors=rng.choice([-1, 1, 2, max(1, n_cand // 3), n_cand, 500]),
            lb=rng.choice([1, 2, 3, 5, 8, 20, 73, 1000]),
            excl_scopes=tuple(rng.sample(scopes, rng.randint(0, 2))),
            incl_scopes=tuple(rng.sample(scopes, rng.randint(0, 1)))))
    return out


def planner_fixtures():
    out = {}
    for name in list(UNET_CONFIGS) + list(CHAIN_CONFIGS):
        g = build(name)
        tg = expand_training_graph(g)
        rec = {
            "forward_sha": sha(dumps_canonical(graph_to_obj(g))),
            "training_sha": sha(dumps_canonical(training_to_obj(tg))),
            "n_nodes": len(g.nodes), "n_tensors": len(g.tensors),
            "serial_order": list(tg.serial_order),
            "cross_phase": cross_phase_tensors(tg),
            "noswap_peak": static_peak_estimate(tg).peak_bytes,
            "cases": [],
        }
        cfgs = [("preset:" + p, dict(n_tensors=PRESETS[p].n_tensors, lb=PRESETS[p].lb,
                                     excl_scopes=PRESETS[p].excl_scopes,
                                     incl_scopes=PRESETS[p].incl_scopes))
                for p in sorted(PRESETS)]
        cfgs += [(f"random{i}", c) for i, c in
                 enumerate(random_cfgs(tg, sum(map(ord, name)) * 7919, 6))]
        for label, kw in cfgs:
            cfg = RewriteConfig(mode="swap", **kw)
            sel = select_swap_tensors(tg, cfg)
            rw, plan = apply_rewrite(tg, cfg)
            pj = plan.to_json()
            case = {"label": label, "cfg": {k: list(v) if isinstance(v, tuple) else v
                                            for k, v in kw.items()},
                    "selection": sel, "plan_sha": sha(pj),
                    "rewritten_sha": sha(dumps_canonical(training_to_obj(rw))),
                    "peak": static_peak_estimate(rw, plan).peak_bytes,
                    "peak_position": static_peak_estimate(rw, plan).peak_position}
            if name in ("toy8", "tiny", "chain5", "f192_bf16") or label == "preset:paper-c4":
                case["plan_json"] = pj
            rec["cases"].append(case)
        for policy in ("speed", "sqrt_n"):
            cfg = RewriteConfig(mode="recompute", ckpt_policy=policy)
            rw, plan = apply_rewrite(tg, cfg)
            rec["cases"].append({
                "label": "recompute:" + policy, "cfg": {"mode": "recompute",
                                                        "ckpt_policy": policy},
                "plan_sha": sha(plan.to_json()),
                "rewritten_sha": sha(dumps_canonical(training_to_obj(rw))),
                "peak": static_peak_estimate(rw, plan).peak_bytes})
        out[name] = rec
    return out


SIM_CASES = [
    # (graph, preset or None, SimConfig kwargs)
    ("toy8", "paper-c1", dict(compute_rate=100.0, d2h_bw=1e6, h2d_bw=1e6)),
    ("toy8", "paper-c4", dict(compute_rate=100.0, d2h_bw=1e6, h2d_bw=1e6)),
    ("tiny", "paper-c1", dict(compute_rate=1e9, d2h_bw=1e8, h2d_bw=1e8, xfer_latency=1e-6)),
    ("tiny", "paper-c3", dict(compute_rate=1e9, d2h_bw=1e8, h2d_bw=1e8)),
    ("chain9_mixed", "paper-c1", dict(compute_rate=1.0, d2h_bw=900.0, h2d_bw=700.0)),
    ("f192_bf16", None, dict(compute_rate=1.35e15, d2h_bw=55e9, h2d_bw=55e9)),
    ("f192_bf16", "paper-c1", dict(compute_rate=1.35e15, d2h_bw=55e9, h2d_bw=55e9)),
    ("f192_bf16", "paper-c4", dict(compute_rate=1.35e15, d2h_bw=55e9, h2d_bw=55e9)),
    ("f192", "paper-c4", dict(compute_rate=2e12, d2h_bw=40e9, h2d_bw=40e9, xfer_latency=10e-6)),
    ("tiny", "paper-c4", dict(compute_rate=1e9, d2h_bw=1e8, h2d_bw=1e8, gpu_budget=4_000_000,
                              enforce_budget=True)),
    ("chain9_mixed", None, dict(gpu_budget=10, enforce_budget=True)),
    ("chain9_mixed", None, dict(gpu_budget=1500, enforce_budget=True)),
]


def sim_fixtures():
    rows = []
    for gname, preset, kw in SIM_CASES:
        tg = expand_training_graph(build(gname))
        if preset:
            tg, plan = apply_rewrite(tg, resolve_preset(preset))
        else:
            plan = None
        row = {"graph": gname, "preset": preset, "sim": kw}
        try:
            rep = simulate(tg, plan, SimConfig(**kw))
            row.update(report_sha=sha(rep.to_json()), makespan=rep.makespan,
                       peak_resident=rep.peak_resident, stall=stall_report(rep),
                       n_events=len(rep.events), n_stalls=len(rep.stalls), error="")
            if gname in ("toy8", "chain9_mixed"):
                row["report_json"] = rep.to_json()
        except swapsim.GraphError as exc:
            row.update(error=type(exc).__name__ + ": " + str(exc))
        rows.append(row)
    return rows


NUMERIC_CASES = [
    # (graph, preset or None, seed)
    ("toy8", None, 1), ("toy8", "paper-c1", 1), ("toy8", "paper-c4", 2), ("toy8", None, 3),
    ("chain9_mixed", None, 5), ("chain9_mixed", "paper-c3", 5),
    ("tiny", None, 1), ("tiny", "paper-c4", 1),
]


def numeric_fixtures():
    ref_numeric.MAX_ELEMENTS = 1 << 22   # the reference caps toy tensors at 10k elements
    index = []
    for gname, preset, seed in NUMERIC_CASES:
        tg = expand_training_graph(build(gname))
        plan = None
        if preset:
            tg, plan = apply_rewrite(tg, resolve_preset(preset))
        loss, grads = ref_numeric.run_numeric(tg, plan, seed)
        fname = f"numeric_{gname}_{preset or 'none'}_s{seed}.npz"
        np.savez_compressed(os.path.join(HERE, fname), loss=np.array(loss),
                            **{k.replace(":", "__"): v for k, v in grads.items()})
        index.append({"graph": gname, "preset": preset, "seed": seed, "file": fname,
                      "loss": loss, "grads": sorted(grads)})
    return index


def main():
    with open(os.path.join(HERE, "planner.json"), "w") as fh:
        json.dump(planner_fixtures(), fh, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "sim.json"), "w") as fh:
        json.dump(sim_fixtures(), fh, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "numeric_index.json"), "w") as fh:
        json.dump(numeric_fixtures(), fh, indent=1, sort_keys=True)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
