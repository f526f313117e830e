#!/bin/bash
# Round-2 pass K: n240 b12 forced-swap at a 171 GiB arena (the unswapped step needs 174.2).
timeout 1500 python bench.py --config n240-b12-tuned --budget-gb 171 --no-cpu-baseline --steps 5 > gpurun_out/k_n240.json 2> gpurun_out/k_n240.err
echo "rc=$?"; tail -3 gpurun_out/k_n240.err
python -c "
import json;d=json.loads(open('gpurun_out/k_n240.json').read().strip().splitlines()[-1]);t=d['tuned_plan'];print('n240', d['ms_per_step'], d['exposed_swap_pct'], t['label'], t['predicted_ms'], t['predicted_exposed_pct'], d['swap']['stall_split_s'])"
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
