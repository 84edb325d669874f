#!/bin/bash
# Extra bench lines (profiles/r02_bench_*.json): Qwen pair (configs[2] models, one GPU), batched T=1
mkdir -p gpurun_out/bl
O=gpurun_out/bl
timeout 900 python bench.py --draft qwen2.5-0.5b --target qwen2.5-7b --K 50 --ratio 5 --no-cpu-baseline > $O/qwen.log 2>&1
timeout 900 python bench.py --batch 32 --new-tokens 256 --no-cpu-baseline > $O/batch32.log 2>&1
timeout 900 python bench.py --batch 32 --new-tokens 256 --temperature 1 --no-cpu-baseline > $O/batch32_t1.log 2>&1
echo done > $O/done
