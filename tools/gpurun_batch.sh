# one gpurun call: GPU tests + bench lines (outputs in gpurun_out/)
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t6.log 2>&1; tail -3 gpurun_out/t6.log
for c in f192-c4 f192-noswap f192-tuned f192-tuned-8 f192-rc-speed p128-b2; do
  extra="--no-cpu-baseline"; [ $c = f192-c4 ] && extra=""
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 $extra > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; tail -2 gpurun_out/b_$c.err
done
