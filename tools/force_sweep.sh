#!/bin/bash
echo "== default"; timeout 200 python tools/microbench.py t8 d116 2>&1 | grep -E "==|graph"
echo "== force"; CARD_CLUSTER_FORCE=1 timeout 200 python tools/microbench.py t8 d116 2>&1 | grep -E "==|graph"
echo "== force, AR"; CARD_CLUSTER_FORCE=1 timeout 200 python tools/microbench.py t1 2>&1 | grep -E "==|graph"
