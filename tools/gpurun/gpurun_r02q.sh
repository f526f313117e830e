#!/bin/bash
# Round-2 pass Q: coalesced (smem-staged) k_igemm epilogue.
timeout 1200 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/q_kt.log 2>&1; tail -2 gpurun_out/q_kt.log
P="timeout 120 python tools/kernel_probe.py"
for s in "convt_fwd 1 96 96 96 128 64" "convt_fwd 1 48 48 48 256 128" "convt_fwd 1 24 24 24 512 256" "convt_fwd 1 12 12 12 1024 512" "convt_dgrad 1 96 96 96 128 64" "convt_dgrad 1 48 48 48 256 128"; do $P $s | tail -1; done
timeout 900 python bench.py --config f192-noswap --no-cpu-baseline > gpurun_out/q_noswap.json 2>gpurun_out/q_noswap.err
python -c "
import json;d=json.loads(open('gpurun_out/q_noswap.json').read().strip().splitlines()[-1]);print('noswap', d['ms_per_step'], d['op_ms_per_step'])"
