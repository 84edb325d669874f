#!/bin/bash
# One iteration on the GPU: targeted tests, persistent-forward timeline, draft/target step times (gpurun_out/it/)
mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 600 python -m pytest tests/test_gpu_parity_full.py tests/test_gpu_llm.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python tools/pfwd_trace.py > $O/pfwd_trace.log 2>&1; echo "rc=$?" >> $O/pfwd_trace.log
SHARP=1e6 NEW=128 timeout 300 python tools/step_times.py > $O/step_times.log 2>&1; echo "rc=$?" >> $O/step_times.log
