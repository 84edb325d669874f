#!/bin/bash
echo "== default"; timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
echo "== 1 CTA/SM 110KB"; CARD_CTAS_PER_SM=1 CARD_GEMM_SMEM_KB=110 timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
echo "== 1 CTA/SM 150KB"; CARD_CTAS_PER_SM=1 CARD_GEMM_SMEM_KB=150 timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
echo "== verify 1 CTA/SM 110KB"; CARD_CTAS_PER_SM=1 CARD_GEMM_SMEM_KB=110 timeout 200 python tools/microbench.py t8 2>&1 | grep -E "graph"
echo "== verify 2 CTA/SM 80KB"; CARD_CTAS_PER_SM=2 CARD_GEMM_SMEM_KB=80 timeout 200 python tools/microbench.py t8 2>&1 | grep -E "graph"
