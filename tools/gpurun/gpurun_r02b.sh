#!/bin/bash
# Round-2 second GPU pass: no-swap op breakdown, forced-budget tuned plans, wgrad/convT probes.
B="timeout 900 python bench.py --no-cpu-baseline --steps 10"
$B --config f192-noswap --op-dump gpurun_out/ops_noswap.json > gpurun_out/b_noswap.json 2> gpurun_out/b_noswap.err
for g in 11 10 8; do
  $B --config f192-tuned --budget-gb $g > gpurun_out/b_tuned_$g.json 2> gpurun_out/b_tuned_$g.err
done
P="timeout 120 python tools/kernel_probe.py"
for s in "conv_wgrad 1 192 192 192 64 64" "conv_wgrad 1 192 192 192 128 64 64" "conv_wgrad 1 96 96 96 256 128 128" "conv_wgrad 1 96 96 96 128 128" "conv_wgrad 1 96 96 96 64 128" "conv_wgrad 1 48 48 48 256 256" "conv_wgrad 1 48 48 48 512 256 256" "conv_wgrad 1 24 24 24 512 512" "conv_wgrad 1 12 12 12 1024 1024" \
         "convt_fwd 1 96 96 96 128 64" "convt_fwd 1 48 48 48 256 128" "convt_fwd 1 24 24 24 512 256" "convt_fwd 1 12 12 12 1024 512" \
         "convt_wgrad 1 96 96 96 128 64" "convt_wgrad 1 48 48 48 256 128" "convt_dgrad 1 96 96 96 128 64" "convt_dgrad 1 48 48 48 256 128"; do
  $P $s >> gpurun_out/probes.txt 2>&1
done
cat gpurun_out/probes.txt
for f in gpurun_out/b_*.json; do echo $f; tail -c 600 $f; echo; done
