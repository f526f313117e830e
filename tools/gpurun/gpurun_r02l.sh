#!/bin/bash
# Round-2 final pass: GPU suite + smoke, every bench config, reference arm, launch list.
mkdir -p gpurun_out/l
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/l/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/l/gputest.log; tail -3 gpurun_out/l/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/l/smoke.log 2>&1; tail -1 gpurun_out/l/smoke.log
timeout 1200 python bench.py > gpurun_out/l/b_default.json 2> gpurun_out/l/b_default.err; tail -c 300 gpurun_out/l/b_default.json
timeout 900 python bench.py --impl reference > gpurun_out/l/b_reference.json 2> gpurun_out/l/b_reference.err
for c in f192-noswap p128-b2 f192-tuned f192-tuned-10 f192-tuned-8 f192-rc-speed f192-rc-sqrt f192-c1; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/l/b_$c.json 2> gpurun_out/l/b_$c.err
  echo "$c rc=$?"
done
timeout 1500 python bench.py --config n240-b12-tuned --no-cpu-baseline --steps 5 > gpurun_out/l/b_n240-b12-tuned.json 2> gpurun_out/l/b_n240-b12-tuned.err; echo "n240 rc=$?"
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-elided-variant > gpurun_out/l/plain.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/l/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-elided-variant > gpurun_out/l/ncu_launch.log 2>&1
echo "launch list rc=$?"
