mkdir -p gpurun_out/bt
timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_gpu_llm.py tests/test_gpu_paging.py -q --timeout 300 --timeout-method=thread > gpurun_out/bt/tests.log 2>&1; echo "rc=$?" >> gpurun_out/bt/tests.log
BS=1,8,16,32,64 timeout 1500 python tools/batch_sweep.py > gpurun_out/bt/sweep.log 2>&1
