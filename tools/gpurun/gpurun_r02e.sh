#!/bin/bash
# Round-2 pass E: exact sub-pixel convT correctness + speed; ncu of the halo-view wgrad and
# the sub-pixel convT kernels.
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "convt" > gpurun_out/e_kt.log 2>&1; tail -3 gpurun_out/e_kt.log
P="timeout 120 python tools/kernel_probe.py"
for s in "convt_fwd 1 96 96 96 128 64" "convt_fwd 1 48 48 48 256 128" "convt_fwd 1 24 24 24 512 256" "convt_fwd 1 12 12 12 1024 512"; do
  echo "new:  $($P $s 2>&1 | tail -1)" >> gpurun_out/e_probes.txt
  echo "old:  $(US_CONVT_CLASSES=1 $P $s 2>&1 | tail -1)" >> gpurun_out/e_probes.txt
done
cat gpurun_out/e_probes.txt
mkdir -p gpurun_out/ncu2
run() {   # name regex probe-args...
  local name=$1 rx=$2; shift 2
  timeout 120 python tools/kernel_probe.py "$@" > gpurun_out/ncu2/$name.plain 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$rx" -c 1 \
    -o gpurun_out/ncu2/$name python tools/kernel_probe.py "$@" > gpurun_out/ncu2/$name.log 2>&1
  echo "$name rc=$? $(tail -1 gpurun_out/ncu2/$name.plain)"
}
run hv_xa_64_64 '^k_wgrad_hv$' conv_wgrad 1 192 192 192 64 64
run hv_xb_256_128 '^k_wgrad_hv$' conv_wgrad 1 96 96 96 256 128 128
run ct_fwd_l0 '^k_igemm$' convt_fwd 1 96 96 96 128 64
run ct_fwd_l1 '^k_igemm$' convt_fwd 1 48 48 48 256 128
run wg_halo_pair_128_64 '^k_wgrad_halo$' conv_wgrad 1 192 192 192 128 64 64
