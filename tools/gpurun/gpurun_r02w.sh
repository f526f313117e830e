#!/bin/bash
# Round-2 pass W: Cout-64 sub-pixel convT with per-tap class runs (no zero-block MMAs).
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "convt" > gpurun_out/w_t.log 2>&1; tail -2 gpurun_out/w_t.log
P="timeout 120 python tools/kernel_probe.py convt_fwd 1 96 96 96 128 64"
echo "runs:  $($P | tail -1)"
echo "full:  $(US_CONVT_RUNS=0 $P | tail -1)"
echo "runs:  $($P | tail -1)"
echo "full:  $(US_CONVT_RUNS=0 $P | tail -1)"
