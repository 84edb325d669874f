#!/bin/bash
# End-of-round pass on one B200: GPU tests, smoke, the default bench line (with the CPU
# baseline), the extra bench lines, the ncu launch list.  Outputs under gpurun_out/final/.
O=gpurun_out/final
mkdir -p $O gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_serial.log 2>&1
timeout 900 python bench.py --temperature 1 --no-cpu-baseline > $O/bench_t1.log 2>&1
timeout 900 python bench.py --bias-sharpness 0 --no-cpu-baseline > $O/bench_s0.log 2>&1
timeout 900 python bench.py --draft qwen2.5-0.5b --target qwen2.5-7b --K 50 --ratio 5 --no-cpu-baseline > $O/bench_qwen.log 2>&1
timeout 900 python bench.py --batch 32 --new-tokens 256 --no-cpu-baseline > $O/bench_batch32.log 2>&1
timeout 900 python bench.py --batch 32 --new-tokens 256 --temperature 1 --no-cpu-baseline > $O/bench_batch32_t1.log 2>&1
echo done > $O/done
