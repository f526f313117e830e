#!/bin/bash
# Round-2 third GPU pass: tuner calibration dump, sqrt_n recompute op breakdown, PCIe
# probe, then ncu --set full of the weight-gradient and transposed-conv kernels.
mkdir -p gpurun_out/ncu
timeout 300 python tools/dump_slots.py 192 192 192 1 gpurun_out/slots_f192.json > gpurun_out/slots.log 2>&1; tail -1 gpurun_out/slots.log
timeout 300 python tools/dump_slots.py 160 240 240 8 gpurun_out/slots_n240b8.json > gpurun_out/slots_n240.log 2>&1; tail -1 gpurun_out/slots_n240.log
timeout 600 python bench.py --config f192-rc-sqrt --steps 5 --no-cpu-baseline --op-dump gpurun_out/ops_rcsqrt.json > gpurun_out/b_rcsqrt.json 2> gpurun_out/b_rcsqrt.err; tail -c 400 gpurun_out/b_rcsqrt.json
timeout 300 python tools/pcie_probe.py 1 > gpurun_out/pcie.json 2>&1; cat gpurun_out/pcie.json
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1; lscpu > gpurun_out/lscpu.txt 2>&1
P="python tools/kernel_probe.py"
run() {   # name regex probe-args...
  local name=$1 rx=$2; shift 2
  timeout 120 $P "$@" > gpurun_out/ncu/$name.plain 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -c 1 \
    -o gpurun_out/ncu/$name $P "$@" > gpurun_out/ncu/$name.log 2>&1
  echo "$name rc=$? $(cat gpurun_out/ncu/$name.plain)"
}
run wg_256_128_96 'k_wgrad<' conv_wgrad 1 96 96 96 256 128 128
run wg_64_64_192 'k_wgrad_halo<' conv_wgrad 1 192 192 192 64 64
run wg_128_128_96 'k_wgrad_halo_a' conv_wgrad 1 96 96 96 128 128
run ct_fwd_l0 'k_igemm<' convt_fwd 1 96 96 96 128 64
run ct_fwd_l3 'k_igemm' convt_fwd 1 12 12 12 1024 512
run ct_wg_l0 'k_wgrad<' convt_wgrad 1 96 96 96 128 64
