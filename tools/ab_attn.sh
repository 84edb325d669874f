mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_gpu_parity_full.py tests/test_gpu_batch.py tests/test_gpu_paging.py -q --timeout 300 --timeout-method=thread > gpurun_out/ab/tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab/tests.log
timeout 300 python tools/attn_tree_probe.py 1000 10 > gpurun_out/ab/attn_new.log 2>&1
cp abtest/base.so paper_2508_04462_b200/libcard_b200.so
timeout 300 python tools/attn_tree_probe.py 1000 10 > gpurun_out/ab/attn_base.log 2>&1
cp abtest/new.so paper_2508_04462_b200/libcard_b200.so
bash tools/ab_so.sh base new > gpurun_out/ab/ab.log 2>&1
