#!/bin/bash
# Round-2 pass V: Chrome traces (reference emit_trace schema) of measured steps.
mkdir -p gpurun_out/v
timeout 900 python bench.py --no-cpu-baseline --no-elided-variant --steps 5 --trace gpurun_out/v/trace_f192-c4.json > gpurun_out/v/b_c4.json 2> gpurun_out/v/b_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --config f192-tuned --no-cpu-baseline --steps 5 --trace gpurun_out/v/trace_f192-tuned.json > gpurun_out/v/b_tuned.json 2> gpurun_out/v/b_tuned.err; echo "tuned rc=$?"
ls -la gpurun_out/v
