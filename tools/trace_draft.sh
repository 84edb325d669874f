#!/bin/bash
for shape in "3072 2048 116 0" "2048 2048 116 1" "16384 2048 116 3" "2048 8192 116 1" "128256 2048 116 0"; do
  timeout 60 python tools/gemm_trace.py $shape 2>&1
done
