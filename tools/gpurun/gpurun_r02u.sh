#!/bin/bash
# Round-2 pass U: full GPU suite (new tuned-plan / forced-budget tests), smoke, default
# bench (link roofline) and reference arm.
mkdir -p gpurun_out/u
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/u/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/u/gputest.log; tail -4 gpurun_out/u/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/u/smoke.log 2>&1; tail -1 gpurun_out/u/smoke.log
timeout 1200 python bench.py > gpurun_out/u/b_default.json 2> gpurun_out/u/b_default.err
python -c "
import json;d=json.loads(open('gpurun_out/u/b_default.json').read().strip().splitlines()[-1]);print('c4', d['ms_per_step'], d['e2e']['value'], d['link_roofline'], d['roofline']['frac'], d['roofline']['frac_of_burst'])"
timeout 900 python bench.py --impl reference > gpurun_out/u/b_reference.json 2> gpurun_out/u/b_reference.err; tail -c 200 gpurun_out/u/b_reference.json
