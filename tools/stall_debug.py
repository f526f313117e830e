"""Which slots of a swapped step stall, and what those slots enqueue."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07816_b200._native import OP
from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer

order = sys.argv[1] if len(sys.argv) > 1 else "need"
INV = {v: k[len("US_OP_"):] for k, v in OP.items() if k.startswith("US_OP_")}
tr = UNetTrainer(TrainConfig(dims=(192, 192, 192), preset="paper-c4", d2h_order=order, graph=False))
x, y = tr.synthetic_batch(seed=0)
tr.load_batch(x, y)
for _ in range(3):
    tr.step()
rep = tr.timeline()
print("step", rep.makespan)
for name, kind, d in sorted(rep.stalls, key=lambda s: -s[2])[:8]:
    print("stall %-30s %.1f ms" % (name, 1e3 * d))
pr = tr.program
names = {d.tid: d.name for d in pr.tensors.values()}
worst = max(rep.stalls, key=lambda s: s[2])[0]
slot = None
inside = False
for code, tids, ia, fa in pr.ops:
    op = INV[code]
    if op == "SLOT_BEGIN":
        inside = pr.slot_names.get(ia[0]) == worst
    if inside or (op == "SLOT_END" and pr.slot_names.get(ia[0]) == worst):
        print(" ", op, [names.get(t, t) for t in tids], ia)
