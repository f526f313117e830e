"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python tools/launch_summary.py launches.csv [title] > summary.txt
Times are serialized and cold-cache (ncu replays each launch alone): use the
share of the step, not the absolute."""
import collections
import csv
import sys


def main(path, title=""):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
        rows.append((r["Kernel Name"], v * scale))
    tot = sum(ms for _, ms in rows)
    agg = collections.defaultdict(lambda: [0.0, 0])
    for k, ms in rows:
        agg[k][0] += ms
        agg[k][1] += 1
    if title:
        print(title)
    print(f"{len(rows)} launches, {tot:.2f} ms kernel time in total\n")
    print(f"{'total ms':>10} {'share':>6} {'count':>6}  kernel")
    for k, (ms, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        name = k if len(k) < 90 else k[:87] + "..."
        print(f"{ms:10.2f} {100 * ms / tot:5.1f}% {n:6d}  {name}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
