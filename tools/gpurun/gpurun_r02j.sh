#!/bin/bash
# Round-2 pass J: transposed-conv kernels after the dead-path cleanup; n240 b12 forced swap
# with lb 60 / 80 in the tuner's search.
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "convt" > gpurun_out/j_t.log 2>&1; tail -2 gpurun_out/j_t.log
P="timeout 120 python tools/kernel_probe.py"
for s in "convt_fwd 1 96 96 96 128 64" "convt_fwd 1 24 24 24 512 256" "convt_fwd 1 12 12 12 1024 512"; do $P $s | tail -1; done
timeout 1500 python bench.py --config n240-b12-tuned --no-cpu-baseline --steps 5 > gpurun_out/j_n240.json 2> gpurun_out/j_n240.err
python -c "
import json;d=json.loads(open('gpurun_out/j_n240.json').read().strip().splitlines()[-1]);t=d['tuned_plan'];print('n240', d['ms_per_step'], d['exposed_swap_pct'], t['label'], t['predicted_ms'], t['predicted_exposed_pct'])"
