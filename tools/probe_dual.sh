#!/bin/bash
# Dual-source (never materialised concat) vs materialised input for the synthesis conv1s.
P="python tools/kernel_probe.py"
for args in "1 192 192 192 128 64 64" "1 96 96 96 256 128 128" "1 48 48 48 512 256 256" "1 24 24 24 1024 512 512"; do
  set -- $args
  for k in conv_fwd conv_wgrad; do
    $P $k $1 $2 $3 $4 $5 $6
    $P $k $1 $2 $3 $4 $5 $6 $7
  done
done
