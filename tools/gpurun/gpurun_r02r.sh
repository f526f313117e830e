#!/bin/bash
# Round-2 pass R: staged k_igemm epilogue on / off, per-op dump of the no-swap step.
for v in 1 0; do
US_IG_STAGED=$v timeout 900 python bench.py --config f192-noswap --no-cpu-baseline --op-dump gpurun_out/r_ops_$v.json > gpurun_out/r_noswap_$v.json 2>gpurun_out/r_noswap_$v.err
python -c "
import json;d=json.loads(open('gpurun_out/r_noswap_$v.json').read().strip().splitlines()[-1]);print('staged=$v', d['ms_per_step'], {k:v for k,v in d['op_ms_per_step'].items() if 'CONV' in k})"
done
