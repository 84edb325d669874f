#!/bin/bash
mkdir -p gpurun_out/mb
O=gpurun_out/mb
timeout 600 python -m pytest tests/test_gpu_llm.py -v -k "concurrent or mailbox" --timeout 120 --timeout-method=thread > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
