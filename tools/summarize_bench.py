"""Print the key fields of bench.py JSON lines (gpurun_out/b_*.json)."""
import glob
import json
import sys

for f in sorted(sys.argv[1:] or glob.glob("gpurun_out/b_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001
        print(f, "ERR", e)
        continue
    sw = d["swap"]
    print(f"{f}: {d['value']:.4g} vox/s  {d['ms_per_step']:.1f} ms  exposed "
          f"{d['exposed_swap_pct']:.1f}%  plan={d['config']['swap_plan']}  e2e {d['e2e']['value']:.4g}")
    print(f"   moved {sw['d2h_bytes_per_step']/1e9:.2f} GB (planned {sw['planned_swap_bytes']/1e9:.2f},"
          f" byte-for-byte {sw['executed_byte_for_byte']})  arena peak {sw['arena_peak_bytes']/2**30:.2f}"
          f" GiB  phys {sw['physical_peak_bytes']/2**30:.2f} GiB  budget "
          f"{(sw['arena_budget_bytes'] or 0)/2**30:.1f}  conv ms {d['conv_ms_per_step']}"
          f"  roofline {d['roofline']['frac']:.3f}")
    if d.get("tuned_plan"):
        t = d["tuned_plan"]
        print(f"   tuned: {t.get('label')}: predicted {t.get('predicted_ms'):.1f} ms /"
              f" {t.get('predicted_exposed_pct'):.1f}%  measured {t.get('measured_ms'):.1f} ms /"
              f" {t.get('measured_exposed_pct'):.1f}%")
    if d.get("elided_variant"):
        e = d["elided_variant"]
        print(f"   elided variant: {e['ms_per_step']:.1f} ms, {e['exposed_swap_pct']:.1f}%")
    print("   ops", {k: v for k, v in list(d["op_ms_per_step"].items())[:8]})
