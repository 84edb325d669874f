#!/bin/bash
mkdir -p gpurun_out/bt
O=gpurun_out/bt
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
