#!/bin/bash
# Round-2 pass M: ncu of the sub-pixel convT (Cout 64, W' form) and the 256-channel halo conv.
mkdir -p gpurun_out/m
run() {   # name regex probe-args...
  local name=$1 rx=$2; shift 2
  timeout 120 python tools/kernel_probe.py "$@" > gpurun_out/m/$name.plain 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$rx" -c 1 \
    -o gpurun_out/m/$name python tools/kernel_probe.py "$@" > gpurun_out/m/$name.log 2>&1
  echo "$name rc=$? $(tail -1 gpurun_out/m/$name.plain)"
}
run ct_fwd_l0 '^k_igemm$' convt_fwd 1 96 96 96 128 64
run halo256_fwd_48 '^k_igemm_halo$' conv_fwd 1 48 48 48 256 256
du -sh gpurun_out
