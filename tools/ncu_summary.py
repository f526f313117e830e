"""Summarise one or more `ncu --set full` captures as a JSON list (for profiles/): duration,
DRAM bytes, tensor-pipe / shared-memory-feed / L2 utilisation, L2->SM bytes and registers,
with the algorithmic work of the captured launch when given.

    python tools/ncu_summary.py out.json rep1.ncu-rep[:flops[:min_bytes[:label]]] ...
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_s_cold",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed":
        "smem_to_tensor_feed_pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_sm_read_bytes",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
}
SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "s": 1.0, "second": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summarise(rep, flops=None, min_bytes=None, label=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")], "report": rep.split("/")[-1]}
        if label:
            d["label"] = label
        for h, u, v in zip(hdr, units, vals):
            if h in WANT and v not in ("", "n/a"):
                d[WANT[h]] = float(v.replace(",", "")) * SCALE.get(u, 1)
        stalls = {}
        for h, v in zip(hdr, vals):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio") and v not in ("", "n/a"):
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len(
                    "_per_issue_active.ratio")]] = float(v)
        d["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:4])
        if "dram_read_bytes" in d:
            d["dram_bytes"] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0.0)
        if flops:
            d["algorithmic_flops"] = flops
            d["tflops_cold"] = flops / d["duration_s_cold"] / 1e12
        if min_bytes:
            d["algorithmic_min_bytes"] = min_bytes
        out.append(d)
    return out


def main(dest, specs):
    res = []
    for spec in specs:
        parts = spec.split(":")
        rep = parts[0]
        flops = float(parts[1]) if len(parts) > 1 and parts[1] else None
        mb = float(parts[2]) if len(parts) > 2 and parts[2] else None
        label = parts[3] if len(parts) > 3 else None
        res += summarise(rep, flops, mb, label)
    with open(dest, "w") as f:
        json.dump(res, f, indent=1)
    for d in res:
        print(json.dumps({k: d.get(k) for k in ("label", "kernel", "duration_s_cold",
                                                 "tflops_cold", "tensor_pipe_active_pct",
                                                 "smem_to_tensor_feed_pct",
                                                 "l2_throughput_pct")}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
