#!/bin/bash
mkdir -p gpurun_out/it2
O=gpurun_out/it2
timeout 900 python -m pytest tests/test_gpu_llm.py tests/test_gpu_cache.py tests/test_gpu_engine.py tests/test_gpu_batch.py -x -q --durations=5 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
NEW=256 B=16 K=3 BSS=16 timeout 600 python tools/batch_acc_probe.py > $O/acc.log 2>&1
