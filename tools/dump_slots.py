"""Measured per-slot compute seconds of the unswapped step (the tuner's calibration) to a
JSON file, so the engine-aware tuner can be explored on a CPU host.

    python tools/dump_slots.py 192 192 192 1 out.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import measure_link, probe_slot_times  # noqa: E402

d, h, w, b = (int(v) for v in sys.argv[1:5])
slots, pb = probe_slot_times((d, h, w), b, 0)
link = measure_link(0)
with open(sys.argv[5], "w") as f:
    json.dump({"dims": [d, h, w], "batch": b, "probe_batch": pb, "link": link,
               "slots": slots}, f, indent=0, sort_keys=True)
print(f"{len(slots)} slots, {1e3 * sum(slots.values()):.2f} ms compute, link {link}")
