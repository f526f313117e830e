#!/bin/bash
# Round-2 pass O: is the Cout-64 sub-pixel convT bound by its L2 reads?  Single CTA vs CTA pair.
P="python tools/kernel_probe.py convt_fwd 1 96 96 96 128 64"
timeout 120 $P | tail -1
US_CONVT_PAIR=1 timeout 120 $P | tail -1
M=gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed
timeout 300 ncu --metrics $M --clock-control none -k regex:^k_igemm$ -c 1 --csv $P > gpurun_out/o_single.csv 2>&1
US_CONVT_PAIR=1 timeout 300 ncu --metrics $M --clock-control none -k regex:^k_igemm$ -c 1 --csv $P > gpurun_out/o_pair.csv 2>&1
grep -E "k_igemm" gpurun_out/o_single.csv | cut -c1-400 | head -8
grep -E "k_igemm" gpurun_out/o_pair.csv | cut -c1-400 | head -8
