"""Summarise the dominant-kernel ncu capture (tools/ncu_dominant.sh) as
profiles/r01_dominant_kernel.json, the file bench.py reads roofline.traffic from.

usage: python tools/ncu_dominant_json.py gpurun_out/dom/z2_fwd.ncu-rep profiles/r01_z2_fwd.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys

# analysis/l0/conv2: 192^3 voxels x 27 taps x 64 x 64 MACs
FLOPS = 2 * 192 ** 3 * 27 * 64 * 64
# bf16 input read once + output written once (the algorithmic minimum)
MIN_BYTES = 2 * 192 ** 3 * 64 * 2

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_sm_read_bytes",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
}
SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1, "": 1}


def main(rep, dest_rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")],
           "slot": "analysis/l0/conv2 (conv fprop 64->64 at 192^3)",
           "source": f"ncu --set full --clock-control none --import-source on "
                     f"(tools/ncu_dominant.sh), {dest_rep}"}
    for h, u, v in zip(hdr, units, vals):
        if h in WANT:
            out[WANT[h]] = float(v.replace(",", "")) * SCALE.get(u, 1)
    d = out.pop("duration")
    out["duration_s_cold"] = d
    out["dram_bytes"] = out["dram_read_bytes"] + out["dram_write_bytes"]
    out["algorithmic_flops"] = FLOPS
    out["tflops_cold"] = FLOPS / d / 1e12
    out["algorithmic_min_bytes"] = MIN_BYTES
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
