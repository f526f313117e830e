#!/bin/bash
# Round-2 pass N: two prefetch lanes (late prefetches on a second H2D stream).
timeout 900 python -m pytest tests/test_gpu_unet.py tests/test_gpu_toy.py -q -x -p no:cacheprovider > gpurun_out/n_t.log 2>&1; tail -2 gpurun_out/n_t.log
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --no-elided-variant > gpurun_out/n_c4_$i.json 2> gpurun_out/n_c4_$i.err
python -c "
import json;d=json.loads(open('gpurun_out/n_c4_$i.json').read().strip().splitlines()[-1]);print('c4 lanes', d['ms_per_step'], d['exposed_swap_pct'], d['clocks']['sm_mhz'], d['swap']['h2d_busy_s'])"
done
cat > /tmp/one_lane.py <<'PY'
import runpy, sys
import paper_1812_07816_b200.unet as U
U.TrainConfig.prefetch_lanes = False
sys.argv = ['bench.py', '--no-cpu-baseline', '--no-elided-variant']
runpy.run_path('bench.py', run_name='__main__')
PY
for i in 1 2; do
PYTHONPATH=. timeout 900 python /tmp/one_lane.py > gpurun_out/n_c4_one_$i.json 2> gpurun_out/n_c4_one_$i.err
python -c "
import json;d=json.loads(open('gpurun_out/n_c4_one_$i.json').read().strip().splitlines()[-1]);print('c4 one lane', d['ms_per_step'], d['exposed_swap_pct'], d['clocks']['sm_mhz'])"
done
