#!/bin/bash
# Round-2 pass T: budget sweep at 192^3 -- swap-only tuning vs all plans (swap, recompute,
# mixes), predicted vs measured.
mkdir -p gpurun_out/t
for b in 11 10.5 10 9.5 9 8.5 8; do
  for m in swap all; do
    timeout 900 python bench.py --config f192-tuned --budget-gb $b --tune-modes $m --no-cpu-baseline --steps 10 > gpurun_out/t/b_${b}_$m.json 2> gpurun_out/t/b_${b}_$m.err
    echo "$b $m rc=$?"
  done
done
