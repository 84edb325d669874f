#!/bin/bash
for S in 4 8 16; do echo "== S=$S"; CARD_ATTN_S=$S timeout 200 python tools/microbench.py t8 2>&1 | grep -E "graph"; done
CARD_ATTN_S=16 timeout 300 python -m pytest tests/test_gpu_llm.py -q -x -k "bf16 or concurrent" 2>&1 | tail -1
