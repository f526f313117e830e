#!/bin/bash
# Full ncu capture of the dominant conv fprop kernel inside the default bench: the z-pair
# halo kernel's first launch of the step is analysis/l0/conv2 fprop (64 -> 64 at 192^3).
set -e
mkdir -p gpurun_out/dom
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/dom/b.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:k_halo_z2 -s 0 -c 1 -o gpurun_out/dom/z2_fwd \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/dom/ncu.log 2>&1
grep -E 'PROF|WARN' gpurun_out/dom/ncu.log | tail -3
