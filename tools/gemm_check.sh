#!/bin/bash
# GEMM tuning pass: split-K plan traces, forward graph timings, LLM parity tests
mkdir -p gpurun_out
timeout 120 python tools/plan_trace.py d116 > gpurun_out/pt_d.log 2>&1
timeout 120 python tools/plan_trace.py t8 > gpurun_out/pt_t.log 2>&1
timeout 300 python tools/microbench.py t1 t8 d116 > gpurun_out/mb.log 2>&1
timeout 600 python -m pytest tests/test_gpu_llm.py -x -q > gpurun_out/pt_llm.log 2>&1; echo rc=$? >> gpurun_out/pt_llm.log
