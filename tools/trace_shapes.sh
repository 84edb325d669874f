#!/bin/bash
for shape in "3072 2048 116 0" "2048 2048 116 1" "16384 2048 116 3" "2048 8192 116 1" "6144 4096 8 0" "4096 4096 8 1" "28672 4096 8 3" "4096 14336 8 1"; do
  timeout 60 python tools/gemm_trace.py $shape 2>&1
done
