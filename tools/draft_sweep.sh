#!/bin/bash
# split-K sweep of the draft (M=116) GEMM shapes without clusters
mkdir -p gpurun_out
for shape in "3072 2048 116 0" "2048 2048 116 1" "16384 2048 116 3" "2048 8192 116 1"; do
  for sp in 1 2 3 4 6 8 12; do
    CARD_NO_CLUSTER=1 CARD_SPLITS=$sp timeout 60 python tools/gemm_probe.py $shape 3 2>&1 | tail -1 | sed "s/^/splits=$sp /"
  done
done
