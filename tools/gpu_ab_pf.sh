#!/bin/bash
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity_full.py tests/test_gpu_llm.py tests/test_gpu_batch.py tests/test_gpu_paging.py -x -q --timeout 300 --timeout-method=thread > gpurun_out/ab/tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab/tests.log
bash tools/ab_so.sh base new > gpurun_out/ab/ab.log 2>&1
