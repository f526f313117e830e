#!/bin/bash
# Round-2 pass F: full GPU suite on the new kernels, convT mode probes, ncu of the halo-view
# weight gradient (XB) and the CTA-pair tap-pair halo weight gradient (Cout 64).
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/f_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/f_gputest.log; tail -4 gpurun_out/f_gputest.log
P="timeout 120 python tools/kernel_probe.py"
for s in "convt_fwd 1 96 96 96 128 64" "convt_fwd 1 48 48 48 256 128" "convt_fwd 1 24 24 24 512 256" "convt_fwd 1 12 12 12 1024 512"; do
  echo "mode:  $($P $s 2>&1 | tail -1)" >> gpurun_out/f_probes.txt
  echo "class: $(US_CONVT_CLASSES=1 $P $s 2>&1 | tail -1)" >> gpurun_out/f_probes.txt
done
cat gpurun_out/f_probes.txt
mkdir -p gpurun_out/ncu3
run() {   # name regex probe-args...
  local name=$1 rx=$2; shift 2
  timeout 120 python tools/kernel_probe.py "$@" > gpurun_out/ncu3/$name.plain 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$rx" -c 1 \
    -o gpurun_out/ncu3/$name python tools/kernel_probe.py "$@" > gpurun_out/ncu3/$name.log 2>&1
  echo "$name rc=$? $(tail -1 gpurun_out/ncu3/$name.plain)"
}
run hv_xb_256_128 '^k_wgrad_hv$' conv_wgrad 1 96 96 96 256 128 128
run wg_halo_64_64 '^k_wgrad_halo$' conv_wgrad 1 192 192 192 64 64
du -sh gpurun_out
