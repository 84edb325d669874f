mkdir -p gpurun_out/bt
timeout 600 python -m pytest tests/test_gpu_batch.py -q --timeout 300 --timeout-method=thread > gpurun_out/bt/tests.log 2>&1; echo "rc=$?" >> gpurun_out/bt/tests.log
timeout 900 python bench.py --batch 32 --new-tokens 256 --no-cpu-baseline > gpurun_out/bt/b32.log 2>&1
