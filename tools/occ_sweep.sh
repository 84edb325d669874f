#!/bin/bash
# forward-graph timing under GEMM occupancy variants (PDL overlap experiment)
echo "== default"; timeout 300 python tools/microbench.py t8 d116 2>&1 | grep -E "graph|GEMMs"
echo "== 1 CTA/SM, 110 KB"; CARD_CTAS_PER_SM=1 CARD_GEMM_SMEM_KB=110 timeout 300 python tools/microbench.py t8 d116 2>&1 | grep -E "graph|GEMMs"
echo "== 1 CTA/SM, 220 KB"; CARD_CTAS_PER_SM=1 timeout 300 python tools/microbench.py t8 d116 2>&1 | grep -E "graph|GEMMs"
echo "== 1 CTA/SM, 110 KB, no PDL"; CARD_PDL=0 CARD_CTAS_PER_SM=1 CARD_GEMM_SMEM_KB=110 timeout 300 python tools/microbench.py t8 2>&1 | grep -E "graph|GEMMs"
