#!/bin/bash
# Round-2 pass I: full GPU suite (poison mode included), then the tiny config under
# compute-sanitizer memcheck (one sanitizer tool per call).
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/i_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/i_gputest.log; tail -3 gpurun_out/i_gputest.log
timeout 300 python tools/sanitize_tiny.py > gpurun_out/i_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 50 python tools/sanitize_tiny.py > gpurun_out/i_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -8 gpurun_out/i_memcheck.log
