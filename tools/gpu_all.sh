#!/bin/bash
mkdir -p gpurun_out/all
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > gpurun_out/all/tests.log 2>&1; echo "rc=$?" >> gpurun_out/all/tests.log
