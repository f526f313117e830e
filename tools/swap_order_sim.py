"""What-if model of the paper-c4 step: D2H issue order FIFO (the reference simulator's)
vs. backward-need priority, with measured no-swap slot times and PCIe bandwidths
(57 / 55 GB/s alone, ~48 GB/s each when both directions are busy)."""
import json
import sys

sys.path.insert(0, ".")
from paper_1812_07816_b200._native import OP
from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer

INV = {v: k[len("US_OP_"):] for k, v in OP.items() if k.startswith("US_OP_")}
trace = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/r31/trace_noswap.json"
dur = {e["name"]: e["dur"] * 1e-6 for e in json.load(open(trace))
       if e.get("ph") == "X" and e["tid"] == 0}
tr = UNetTrainer(TrainConfig(dims=(192, 192, 192), preset="paper-c4"), device_engine=False)
pr = tr.program
names = {d.tid: d.name for d in pr.tensors.values()}
nbytes = {d.tid: d.nbytes for d in pr.tensors.values()}
slot, nslots = None, len(pr.slot_names)
prod, trig, first_read = {}, {}, {}
for code, tids, ia, fa in pr.ops:
    op = INV[code]
    if op == "SLOT_BEGIN":
        slot = ia[0]
    elif op == "SWAP_OUT":
        prod[tids[0]] = slot
    elif op == "SWAP_IN":
        trig[tids[0]] = (ia[1], tids[1])
    elif slot is not None and op not in ("SLOT_END", "FREE", "SWAP_RELEASE"):
        for t in tids:
            if t >= 0 and names[t].endswith("@in") and t not in first_read:
                first_read[t] = slot
src_of_in = {v[1]: k for k, v in trig.items()}
need = {src: first_read[inn] for inn, src in src_of_in.items()}
sdur = [dur.get(pr.slot_names.get(p, "optimizer"), 0.0) for p in range(nslots)]


def simulate(priority):
    dt = 2e-5
    t = 0.0
    p = 0                       # current compute slot
    slot_left = sdur[0]
    slot_end = {}
    d2h_q, d2h_cur, d2h_left, d2h_done = [], None, 0.0, {}
    h2d_q, h2d_cur, h2d_left, h2d_done = [], None, 0.0, {}
    issued = set()
    while p < nslots:
        # compute: a slot may start only when its prefetched inputs arrived
        waits = [inn for inn, s in first_read.items() if s == p and inn not in h2d_done]
        if not waits:
            slot_left -= dt
            if slot_left <= 0:
                slot_end[p] = t
                for src, ps in prod.items():
                    if ps == p:
                        d2h_q.append(src)
                for src, (ts, inn) in trig.items():
                    if ts == p:
                        h2d_q.append(src)
                p += 1
                slot_left = sdur[p] if p < nslots else 0
        both = d2h_cur is not None and h2d_cur is not None
        bw_d, bw_h = (48e9, 48e9) if both else (57e9, 55e9)
        if d2h_cur is None and d2h_q:
            if priority:
                d2h_q.sort(key=lambda s: need[s])
            d2h_cur = d2h_q.pop(0)
            d2h_left = nbytes[d2h_cur]
        if d2h_cur is not None:
            d2h_left -= bw_d * dt
            if d2h_left <= 0:
                d2h_done[d2h_cur] = t
                d2h_cur = None
        if h2d_cur is None and h2d_q and h2d_q[0] in d2h_done:
            h2d_cur = h2d_q.pop(0)
            h2d_left = nbytes[h2d_cur]
        if h2d_cur is not None:
            h2d_left -= bw_h * dt
            if h2d_left <= 0:
                h2d_done[trig[h2d_cur][1]] = t
                h2d_cur = None
        t += dt
    return t


print("compute only %.1f ms" % (1e3 * sum(sdur)))
print("FIFO D2H      %.1f ms" % (1e3 * simulate(False)))
print("priority D2H  %.1f ms" % (1e3 * simulate(True)))
