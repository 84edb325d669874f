#!/bin/bash
# Round profile artefacts -> gpurun_out/prof/ (summarised into profiles/ by tools/make_profiles.py)
set -x
mkdir -p gpurun_out/prof
# 1. launch list of a short CARD + AR decode on the BASELINE config
NEW=32 SHARP=${SHARP:-1e6} timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches_card.csv python tools/profile_steps.py > gpurun_out/prof/launches_card.log 2>&1
# 2. per-launch DRAM traffic of every tc_gemm launch of one target verify forward (M = r+1 = 8)
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:tc_gemm --csv --log-file gpurun_out/prof/traffic_t8.csv python tools/fwd_profile.py t8 > gpurun_out/prof/traffic_t8.log 2>&1
# 3. one full capture of the dominant kernel (the verify forward's gate/up GEMM, tc_gemm<3>)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel -s 2 -c 1 \
  -o gpurun_out/prof/gemm_gu_t8 python tools/gemm_probe.py 28672 4096 8 3 3 > gpurun_out/prof/gemm_gu_t8.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel -s 2 -c 1 \
  -o gpurun_out/prof/gemm_qkv_d116 python tools/gemm_probe.py 3072 2048 116 0 3 > gpurun_out/prof/gemm_qkv_d116.log 2>&1
