#!/bin/bash
for S in 8 4 2 4 8; do echo "== draft S=$S"; CARD_ATTN_S=$S timeout 200 python tools/microbench.py d116 2>&1 | grep -E "graph replay"; done
