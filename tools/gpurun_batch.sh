set -x
bash tools/probe_dual.sh > gpurun_out/dual.log 2>&1; cat gpurun_out/dual.log
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_unet.py -k "dual or swapping" -q -p no:cacheprovider > gpurun_out/t7.log 2>&1; tail -3 gpurun_out/t7.log
timeout 900 python bench.py --config f192-noswap --steps 10 --no-cpu-baseline --op-dump gpurun_out/ops_dual.json > gpurun_out/b_ns_dual.json 2>&1
timeout 900 python bench.py --config f192-noswap --steps 10 --no-cpu-baseline --no-dual-source --op-dump gpurun_out/ops_mat.json > gpurun_out/b_ns_mat.json 2>&1
timeout 900 python bench.py --config f192-tuned-8 --steps 10 --no-cpu-baseline > gpurun_out/b_f192-tuned-8.json 2> gpurun_out/b_f192-tuned-8.err; tail -2 gpurun_out/b_f192-tuned-8.err
