#!/bin/bash
# per-CTA weight streaming rate: bulk-copy piece size, cluster split of the draft down projection
mkdir -p gpurun_out
for p in 1 2 4 8; do echo "== pieces $p"; CARD_BULK_PIECES=$p CARD_SPLITS=4 CARD_CLUSTER_FORCE=1 timeout 120 python tools/gemm_trace.py 2048 8192 16 0 | grep -E "first_kb|last_mma|span"; done
for p in 1 4; do echo "== d116 pieces $p"; CARD_BULK_PIECES=$p timeout 120 python tools/gemm_trace.py 2048 8192 116 1 | grep -E "first_kb|last_mma|span"; done
echo "== d116 S=8 2/SM 112KB"; CARD_CTAS_PER_SM=2 CARD_GEMM_SMEM_KB=112 CARD_SPLITS=8 CARD_CLUSTER_FORCE=1 timeout 120 python tools/gemm_trace.py 2048 8192 116 1 | grep -E "^\{|first_kb|last_mma|done|span"
echo "== d116 S=8 force"; CARD_SPLITS=8 CARD_CLUSTER_FORCE=1 timeout 120 python tools/gemm_trace.py 2048 8192 116 1 | grep -E "^\{|first_kb|last_mma|done|span"
for p in 1 4; do echo "== fwd pieces $p"; CARD_BULK_PIECES=$p timeout 200 python tools/microbench.py t8 d116 | grep "graph replay"; done
