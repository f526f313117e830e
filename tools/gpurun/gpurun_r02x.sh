#!/bin/bash
# Round-2 pass X: weight gradients on a side stream -- exactness, then no-swap and paper-c4
# steps with it off / on.
timeout 900 python -m pytest tests/test_gpu_unet.py -q -x -p no:cacheprovider -k "wgrad_stream or poison or swapping" > gpurun_out/x_t.log 2>&1; tail -2 gpurun_out/x_t.log
for i in 1 2; do
timeout 900 python bench.py --config f192-noswap --no-cpu-baseline > gpurun_out/x_ns_off_$i.json 2>/dev/null
PYTHONPATH=. timeout 900 python tools/bench_wgrad_stream.py --config f192-noswap --no-cpu-baseline > gpurun_out/x_ns_on_$i.json 2>gpurun_out/x_ns_on_$i.err
python -c "
import json
for n in ('off','on'):
    d=json.loads(open('gpurun_out/x_ns_%s_$i.json'%n).read().strip().splitlines()[-1]); print('noswap', n, d['ms_per_step'], d['clocks']['sm_mhz'])"
done
timeout 900 python bench.py --no-cpu-baseline --no-elided-variant > gpurun_out/x_c4_off.json 2>/dev/null
PYTHONPATH=. timeout 900 python tools/bench_wgrad_stream.py --no-cpu-baseline --no-elided-variant > gpurun_out/x_c4_on.json 2>gpurun_out/x_c4_on.err
python -c "
import json
for n in ('off','on'):
    d=json.loads(open('gpurun_out/x_c4_%s.json'%n).read().strip().splitlines()[-1]); print('c4', n, d['ms_per_step'], d['clocks']['sm_mhz'])"
