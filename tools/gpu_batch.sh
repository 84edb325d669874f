#!/bin/bash
mkdir -p gpurun_out/bt
O=gpurun_out/bt
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
BS=1,2,4,8,16,32,64 timeout 1500 python tools/batch_sweep.py > $O/sweep.log 2>&1; echo "rc=$?" >> $O/sweep.log
