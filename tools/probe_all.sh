#!/bin/bash
# per-kernel timings of the production conv shapes (192^3 U-Net, base 64)
P="python tools/kernel_probe.py"
for k in conv_fwd conv_dgrad conv_wgrad; do
  $P $k 1 192 192 192 64 64
  $P $k 1 96 96 96 128 128
  $P $k 1 48 48 48 256 256
  $P $k 1 24 24 24 512 512
  $P $k 1 12 12 12 1024 1024
done
$P conv_fwd 1 192 192 192 32 64
$P conv_wgrad 1 192 192 192 32 64
$P conv_fwd 1 192 192 192 128 64
$P conv_dgrad 1 192 192 192 128 64
$P conv_wgrad 1 192 192 192 128 64
for k in convt_fwd convt_dgrad convt_wgrad; do
  $P $k 1 96 96 96 128 64
  $P $k 1 12 12 12 1024 512
done
