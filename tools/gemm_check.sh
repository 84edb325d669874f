#!/bin/bash
# GEMM parity tests + per-shape probe + model microbench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_llm.py -x -q > gpurun_out/gemm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gemm_tests.log
for shape in "3072 2048 116 0" "2048 2048 116 1" "16384 2048 116 3" "2048 8192 116 1" "6144 4096 8 0" "4096 4096 8 1" "28672 4096 8 3" "4096 14336 8 1"; do
  timeout 60 python tools/gemm_probe.py $shape 3 2>&1 | tail -2
done > gpurun_out/probe2.log
timeout 300 python tools/microbench.py t8 d116 > gpurun_out/microbench2.log 2>&1
