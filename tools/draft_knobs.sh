#!/bin/bash
echo "== default"; timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
echo "== 2 CTA/SM"; CARD_CTAS_PER_SM=2 timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
echo "== 2 CTA/SM splits 8"; CARD_CTAS_PER_SM=2 CARD_SPLITS=8 timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
echo "== 1 CTA/SM splits 8"; CARD_SPLITS=8 timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
echo "== 1 CTA/SM splits 2"; CARD_SPLITS=2 timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
