"""Checkpoint/recompute planner (the paper's section-5 alternative to swapping).

Drop-in for the recompute half of ``pkg/src/swapsim/rewrite.py``:
``plan_checkpoints`` (rewrite.py:208-234) picks the kept tensors and
``insert_recompute`` (rewrite.py:237-353) splices forward-op clones ahead of
each backward segment.  The plan JSON is byte-identical to the reference's,
and ``unet.py`` lowers every clone ``<f>@rc<s>`` to the same real op as f
(BN clones reuse the forward's saved batch statistics), so a recompute step
on the GPU is bit-identical to the no-swap step (SURVEY.md section 8(f),
item 2; bench configs f192-rc-speed / f192-rc-sqrt).
"""
from __future__ import annotations

import math

from .graph import GraphError, GraphSpec, NodeSpec, TensorDesc
from .training import TrainingGraph, cross_phase_tensors


def plan_checkpoints(tg: TrainingGraph, cfg) -> list[str]:
    from .rewrite import CKPT_KINDS
    cfg.validate()
    if cfg.mode != "recompute":
        raise GraphError(f"plan_checkpoints requires mode 'recompute', got {cfg.mode!r}")
    g = tg.graph
    cands = cross_phase_tensors(tg)
    if cfg.ckpt_policy == "speed":
        keep = {t for t in cands if g.node(g.tensor(t).producer).kind in CKPT_KINDS}
    elif cfg.ckpt_policy == "sqrt_n":
        step = math.ceil(math.sqrt(len(cands))) if cands else 1
        keep = {t for i, t in enumerate(cands, start=1) if i % step == 0}
    else:
        bad = [t for t in cfg.manual_ckpts if t not in set(cands)]
        if bad:
            raise GraphError(f"manual checkpoint {bad[0]!r} is not a cross-phase tensor")
        keep = set(cfg.manual_ckpts)
    cand_set = set(cands)
    for n in g.nodes:
        if n.kind == "loss":
            keep.update(t for t in n.inputs if t in cand_set)
    return sorted(keep, key=lambda t: (tg.position(g.tensor(t).producer), t))


def insert_recompute(tg: TrainingGraph, checkpoints) -> tuple[TrainingGraph, object]:
    from .rewrite import RewritePlan
    g = tg.graph
    cross = set(cross_phase_tensors(tg))
    for t in checkpoints:
        if t not in cross:
            raise GraphError(f"checkpoint {t!r} is not a cross-phase tensor")
    kept = set(checkpoints)
    graph_inputs = {n.outputs[0] for n in g.nodes
                    if n.phase == "forward" and not n.inputs and n.outputs}
    cut = tg.boundary_position + 1
    fwd_ids, bwd_ids = list(tg.serial_order[:cut]), list(tg.serial_order[cut:])

    def resident(tid):
        return tid in kept or tid in graph_inputs

    segment_of, seg = {}, 0
    for nid in fwd_ids:
        segment_of[nid] = seg
        outs = g.node(nid).outputs
        if outs and outs[0] in kept:
            seg += 1

    # Consecutive grads whose forward op lies in the same segment form a group.
    groups: list[list] = []
    for gid in bwd_ids:
        s = segment_of.get(tg.grad_of.get(gid), -1)
        if groups and groups[-1][0] == s:
            groups[-1][1].append(gid)
        else:
            groups.append([s, [gid]])

    by_id = {n.id: n for n in g.nodes}
    tensors = list(g.tensors)
    clones_all: list[NodeSpec] = []
    plan = RewritePlan(mode="recompute", checkpoints=tuple(sorted(kept)))
    serial_bwd: list[str] = []
    for s, gids in groups:
        remap: dict[str, str] = {}
        made: list[str] = []

        def materialize(tid):
            if resident(tid):
                return tid
            if tid in remap:
                return remap[tid]
            prod = g.node(g.tensor(tid).producer)
            if prod.phase != "forward" or prod.kind == "loss":
                return tid
            if not prod.inputs:
                raise GraphError(f"segment needs tensor {tid!r} with no preceding checkpoint "
                                 f"and no graph input to recompute from")
            args = tuple(materialize(x) for x in prod.inputs)
            cid, ctid = f"{prod.id}@rc{s}", f"{tid}@rc{s}"
            src = g.tensor(tid)
            clones_all.append(NodeSpec(id=cid, kind=prod.kind, inputs=args, outputs=(ctid,),
                                       cost_units=prod.cost_units, scope=prod.scope,
                                       phase="backward"))
            tensors.append(TensorDesc(id=ctid, producer=cid, shape=src.shape,
                                      channels=src.channels, elem_bytes=src.elem_bytes,
                                      scope=src.scope))
            plan.clone_map[cid] = prod.id
            made.append(cid)
            remap[tid] = ctid
            return ctid

        for gid in gids:
            node = by_id[gid]
            new_in = []
            for tid in node.inputs:
                fwd_made = (g.has_tensor(tid)
                            and g.node(g.tensor(tid).producer).phase == "forward")
                new_in.append(materialize(tid) if fwd_made and not resident(tid) else tid)
            by_id[gid] = NodeSpec(id=node.id, kind=node.kind, inputs=tuple(new_in),
                                  outputs=node.outputs, cost_units=node.cost_units,
                                  scope=node.scope, phase=node.phase)
        if made:
            first = min(tg.position(plan.clone_map[c]) for c in made)
            anchor = ""
            for nid in reversed(fwd_ids[:first]):
                outs = g.node(nid).outputs
                if outs and outs[0] in kept:
                    anchor = outs[0]
                    break
            plan.recompute_segments += ((anchor, tuple(plan.clone_map[c] for c in made)),)
        serial_bwd += made + gids

    rewritten = GraphSpec(nodes=tuple(by_id[n.id] for n in g.nodes) + tuple(clones_all),
                          tensors=tuple(tensors), control_edges=g.control_edges,
                          metadata=dict(g.metadata))
    return (TrainingGraph(graph=rewritten, reuse_edges=tg.reuse_edges,
                          serial_order=tuple(fwd_ids) + tuple(serial_bwd),
                          grad_of=dict(tg.grad_of)), plan)
