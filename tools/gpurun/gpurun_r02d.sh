#!/bin/bash
# Round-2 pass D: halo-view wgrad correctness + speed, tuned forced-swap configs, sqrt_n fix.
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "wgrad" > gpurun_out/d_kt.log 2>&1; tail -3 gpurun_out/d_kt.log
P="timeout 120 python tools/kernel_probe.py"
for s in "conv_wgrad 1 192 192 192 64 64" "conv_wgrad 1 192 192 192 128 64 64" "conv_wgrad 1 96 96 96 256 128 128" "conv_wgrad 1 96 96 96 128 128" "conv_wgrad 1 96 96 96 64 128" "conv_wgrad 1 48 48 48 256 256" "conv_wgrad 1 48 48 48 512 256 256" "conv_wgrad 1 48 48 48 128 256" "conv_wgrad 1 24 24 24 512 512" "conv_wgrad 1 24 24 24 1024 512 512" "conv_wgrad 1 24 24 24 256 512"; do
  echo "hv:   $($P $s 2>&1 | tail -1)" >> gpurun_out/d_probes.txt
  echo "old:  $(US_NO_HV=1 $P $s 2>&1 | tail -1)" >> gpurun_out/d_probes.txt
done
cat gpurun_out/d_probes.txt
B="timeout 900 python bench.py --no-cpu-baseline --steps 10"
$B --config f192-noswap --op-dump gpurun_out/d_ops_noswap.json > gpurun_out/d_noswap.json 2> gpurun_out/d_noswap.err; tail -c 300 gpurun_out/d_noswap.json
$B --config f192-rc-sqrt > gpurun_out/d_rcsqrt.json 2> gpurun_out/d_rcsqrt.err; tail -c 300 gpurun_out/d_rcsqrt.json
$B --config f192-tuned > gpurun_out/d_tuned11.json 2> gpurun_out/d_tuned11.err; tail -c 300 gpurun_out/d_tuned11.json
$B --config f192-tuned-10 > gpurun_out/d_tuned10.json 2> gpurun_out/d_tuned10.err; tail -c 300 gpurun_out/d_tuned10.json
