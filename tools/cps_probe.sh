for cfg in "" "CARD_CTAS_PER_SM=2 CARD_GEMM_SMEM_KB=118" "CARD_CTAS_PER_SM=2 CARD_GEMM_SMEM_KB=118 CARD_SPLITS=4" "CARD_CTAS_PER_SM=2 CARD_GEMM_SMEM_KB=150 CARD_SPLITS=4"; do
  echo "== [$cfg]"; env $cfg timeout 200 python tools/microbench.py d116 2>&1 | grep -E "GEMM-only|graph replay|Error|error"
done
