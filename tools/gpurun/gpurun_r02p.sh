#!/bin/bash
# Round-2 pass P: source-level stall sampling of the Cout-64 sub-pixel convT.
mkdir -p gpurun_out/p
P="python tools/kernel_probe.py convt_fwd 1 96 96 96 128 64"
timeout 120 $P > gpurun_out/p/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^k_igemm$" -c 1 -o gpurun_out/p/ct $P > gpurun_out/p/ncu.log 2>&1
echo "rc=$?"
