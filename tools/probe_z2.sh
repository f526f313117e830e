#!/bin/bash
# L0 64-channel halo convs: CTA-pair z-pair kernels (default) vs single-CTA (US_NO_Z2_PAIR=1).
P="python tools/kernel_probe.py"
for v in 0 1; do
  echo "US_NO_Z2_PAIR=$v"
  US_NO_Z2_PAIR=$v $P conv_fwd 1 192 192 192 64 64
  US_NO_Z2_PAIR=$v $P conv_fwd 1 192 192 192 128 64
  US_NO_Z2_PAIR=$v $P conv_dgrad 1 192 192 192 64 64
  US_NO_Z2_PAIR=$v $P conv_dgrad 1 96 96 96 64 128
done
for v in 0 1; do
  echo "128 channels US_NO_Z2_PAIR=$v"
  US_NO_Z2_PAIR=$v $P conv_fwd 1 96 96 96 128 128
  US_NO_Z2_PAIR=$v $P conv_dgrad 1 96 96 96 128 128
  US_NO_Z2_PAIR=$v $P conv_dgrad 1 192 192 192 128 64
done
for v in 0 1; do
  echo "wgrad 128->64 US_NO_Z2_PAIR=$v"
  US_NO_Z2_PAIR=$v $P conv_wgrad 1 192 192 192 128 64
done
