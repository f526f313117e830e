"""Timeline invariants of the reference's property suite (props.py:71-130), restated for
measured GPU timelines -- TEST INFRASTRUCTURE ONLY."""
from paper_1812_07816_b200.graph import tensor_bytes

EPS = 2e-6   # event timestamps have ~0.5 us resolution


def event_map(report):
    return {nid: (s, e) for nid, _, s, e in report.events}


def dependency_violations(tg, report):
    """props.py:71-77: every data edge u->v has end(u) <= start(v)."""
    ev = event_map(report)
    bad = []
    for u, v in tg.graph.edges():
        if u in ev and v in ev and ev[u][1] > ev[v][0] + EPS:
            bad.append(f"edge {u}->{v}: end {ev[u][1]:.6f} > start {ev[v][0]:.6f}")
    return bad


def swap_violations(tg, plan, report, elided=()):
    """props.py:118-130: a swap-out starts after its producer ends; a swap-in ends before
    its earliest consumer starts.  `elided`: planned swaps the engine skipped (dead BN
    outputs) -- they have no copy events."""
    g = tg.graph
    ev = event_map(report)
    bad = []
    for tid, (out_id, in_id, _) in sorted(plan.swapped.items()):
        if tid in elided:
            continue
        producer = g.tensor(tid).producer
        if ev[out_id][0] < ev[producer][1] - EPS:
            bad.append(f"swap_out of {tid} starts before its producer ends")
        starts = [ev[c][0] for c in g.consumers(g.node(in_id).outputs[0]) if c in ev]
        if starts and ev[in_id][1] > min(starts) + EPS:
            bad.append(f"swap_in of {tid} finishes after its earliest consumer starts")
    return bad


def resident_never_negative(tg, report):
    """props.py:80-116 (derived residency trace): bytes never go negative."""
    g = tg.graph
    ev = event_map(report)
    delta = {}
    for t in g.tensors:
        if t.producer not in ev:
            continue
        ends = [ev[c][1] for c in g.consumers(t.id) if c in ev]
        a, b = ev[t.producer][0], (max(ends) if ends else ev[t.producer][1])
        delta[a] = delta.get(a, 0) + tensor_bytes(t)
        delta[b] = delta.get(b, 0) - tensor_bytes(t)
    cur = 0
    for when in sorted(delta):
        cur += delta[when]
        if cur < 0:
            return False
    return True
