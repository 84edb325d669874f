#!/bin/bash
# split-K / occupancy calibration sweep for the weight-streaming GEMM
for shape in "28672 4096 8 3" "4096 4096 8 1" "4096 14336 8 1" "6144 4096 8 0" "128256 4096 8 0" "16384 2048 116 3" "3072 2048 116 0" "2048 8192 116 1"; do
  for cps in 1 2; do
    for sp in 1 2 3 4 6 8 12 16; do
      CARD_CTAS_PER_SM=$cps CARD_SPLITS=$sp python tools/gemm_probe.py $shape 3 2>/dev/null | tail -1 | sed "s/^/cps=$cps splits=$sp /"
    done
  done
done
