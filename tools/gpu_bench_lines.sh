#!/bin/bash
# Extra bench lines (profiles/r02_bench_*.json): batched configs[4], pure random-init (s=0), T=1
mkdir -p gpurun_out/bl
O=gpurun_out/bl
timeout 900 python bench.py --no-cpu-baseline > $O/serial.log 2>&1
timeout 900 python bench.py --batch 32 --new-tokens 256 --no-cpu-baseline > $O/batch32.log 2>&1
timeout 900 python bench.py --batch 8 --new-tokens 256 --no-cpu-baseline > $O/batch8.log 2>&1
timeout 900 python bench.py --bias-sharpness 0 --no-cpu-baseline > $O/s0.log 2>&1
timeout 900 python bench.py --temperature 1 --no-cpu-baseline > $O/t1.log 2>&1
echo done > $O/done
