#!/bin/bash
# Full round pass on one B200: parity tests, smoke, bench lines (serial /
# concurrent, T=0 / T=1, Llama / Qwen), forward microbench and timelines.
mkdir -p gpurun_out/round
O=gpurun_out/round
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_serial.log 2>&1
timeout 900 python bench.py --mode concurrent --no-cpu-baseline > $O/bench_concurrent.log 2>&1
timeout 900 python bench.py --temperature 1 --no-cpu-baseline > $O/bench_t1_serial.log 2>&1
timeout 900 python bench.py --temperature 1 --mode concurrent --no-cpu-baseline > $O/bench_t1_concurrent.log 2>&1
timeout 900 python bench.py --draft qwen2.5-0.5b --target qwen2.5-7b --K 50 --ratio 5 --no-cpu-baseline > $O/bench_qwen_serial.log 2>&1
timeout 900 python bench.py --draft qwen2.5-0.5b --target qwen2.5-7b --K 50 --ratio 5 --mode concurrent --no-cpu-baseline > $O/bench_qwen_concurrent.log 2>&1
timeout 600 python tools/microbench.py t1 t8 d116 > $O/microbench.log 2>&1
timeout 300 python tools/graph_timeline.py d116 > $O/timeline_draft.log 2>&1
timeout 300 python tools/graph_timeline.py t8 > $O/timeline_verify.log 2>&1
echo done > $O/done
