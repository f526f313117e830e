#!/bin/bash
# Full ncu capture of the dominant conv fprop kernel (L0 halo N=64: the first halo launch of the step is analysis/l0/conv2 fprop) inside the default bench.
set -e
mkdir -p gpurun_out/r48
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r48/b.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:k_igemm_halo -s 0 -c 1 -o gpurun_out/r48/halo64_fwd \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r48/ncu.log 2>&1
grep -E 'PROF|WARN' gpurun_out/r48/ncu.log | tail -3
