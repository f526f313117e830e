#!/bin/bash
# L0 N=64 halo convs: z-pair kernel (default) vs the 8x16x1 halo kernel (US_NO_Z2=1).
for z in 0 1; do
  echo "US_NO_Z2=$z"
  US_NO_Z2=$z bash tools/probe_l0.sh
done
