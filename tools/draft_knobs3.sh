#!/bin/bash
echo "== default"; timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
echo "== 2 CTA/SM (110KB)"; CARD_CTAS_PER_SM=2 timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
echo "== 1 CTA/SM forced clusters"; CARD_CLUSTER_FORCE=1 timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph"
