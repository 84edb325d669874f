#!/bin/bash
# Round profile artefacts -> gpurun_out/prof/ (summarised into profiles/ by tools/make_profiles.py rNN)
set -x
mkdir -p gpurun_out/prof
P=gpurun_out/prof
# 1. launch list of a short CARD + AR decode on the BASELINE config (the bench's request)
NEW=32 SHARP=${SHARP:-1e6} timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $P/launches_card.csv python tools/profile_steps.py > $P/launches_card.log 2>&1
# 2. per-launch DRAM traffic of every tc_gemm launch of one target verify forward (M = r+1 = 8)
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:tc_gemm --csv --log-file $P/traffic_t8.csv python tools/fwd_profile.py t8 > $P/traffic_t8.log 2>&1
# 3. full captures: the verify's gate/up GEMM, the draft's persistent layer kernel, its tree attention,
#    and the fused lm_head + softmax + top-k of the draft step
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel -s 2 -c 1 \
  -o $P/gemm_gu_t8 python tools/gemm_probe.py 28672 4096 8 3 3 > $P/gemm_gu_t8.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pfwd_kernel -s 40 -c 1 \
  -o $P/pfwd_d116 python tools/fwd_profile.py d116 > $P/pfwd_d116.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc_kernel -s 40 -c 1 \
  -o $P/attn_tc_d116 python tools/fwd_profile.py d116 > $P/attn_tc_d116.log 2>&1
NEW=8 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name-base demangled -k "regex:tc_gemm_kernel<.int.5" -s 2 -c 1 \
  -o $P/lmhead_topk python tools/profile_steps.py > $P/lmhead_topk.log 2>&1
echo done > $P/done
