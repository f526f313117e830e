#!/bin/bash
# Round-2 pass H: CTA-pair sub-pixel convT (Cout 64) and the look-ahead swap-out order.
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_unet.py -q -x -p no:cacheprovider -k "convt or swap or c4 or timeline" > gpurun_out/h_t.log 2>&1; tail -3 gpurun_out/h_t.log
P="timeout 120 python tools/kernel_probe.py"
echo "pair:   $($P convt_fwd 1 96 96 96 128 64 | tail -1)"
echo "single: $(US_NO_Z2_PAIR=1 $P convt_fwd 1 96 96 96 128 64 | tail -1)"
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --no-elided-variant > gpurun_out/h_c4_$i.json 2> gpurun_out/h_c4_$i.err; python -c "
import json;d=json.loads(open('gpurun_out/h_c4_$i.json').read().strip().splitlines()[-1]);print('c4', d['ms_per_step'], d['exposed_swap_pct'], d['swap']['physical_peak_bytes']/2**30, d['clocks']['sm_mhz'], d['op_ms_per_step'].get('CONVT_FWD'))"
done
