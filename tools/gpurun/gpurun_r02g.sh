#!/bin/bash
# Round-2 pass G: bench lines of every config, reference arm, launch list and the dominant
# kernel capture of the default command.
mkdir -p gpurun_out/g
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/g/smi.txt 2>&1
timeout 1200 python bench.py > gpurun_out/g/b_default.json 2> gpurun_out/g/b_default.err; tail -c 400 gpurun_out/g/b_default.json
timeout 900 python bench.py --impl reference > gpurun_out/g/b_reference.json 2> gpurun_out/g/b_reference.err; tail -c 300 gpurun_out/g/b_reference.json
for c in f192-noswap p128-b2 f192-tuned f192-tuned-10 f192-tuned-8 f192-rc-speed f192-rc-sqrt f192-c1; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/g/b_$c.json 2> gpurun_out/g/b_$c.err
  echo "$c rc=$? $(tail -c 200 gpurun_out/g/b_$c.json)"
done
timeout 1500 python bench.py --config n240-b12-tuned --no-cpu-baseline --steps 5 > gpurun_out/g/b_n240-b12-tuned.json 2> gpurun_out/g/b_n240-b12-tuned.err
echo "n240 rc=$? $(tail -c 300 gpurun_out/g/b_n240-b12-tuned.json)"; tail -3 gpurun_out/g/b_n240-b12-tuned.err
# launch list of the default command (serialised, cold: shares, not absolutes)
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-elided-variant > gpurun_out/g/plain.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/g/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-elided-variant > gpurun_out/g/ncu_launch.log 2>&1
echo "launch list rc=$? $(wc -l < gpurun_out/g/launches_c4.csv)"
# dominant conv fprop kernel, full set
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:^k_halo_z2$" -s 0 -c 1 \
  -o gpurun_out/g/z2_fwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-elided-variant > gpurun_out/g/ncu_dom.log 2>&1
echo "dominant rc=$?"; du -sh gpurun_out
