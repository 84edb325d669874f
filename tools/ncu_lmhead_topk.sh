mkdir -p gpurun_out/prof
NEW=8 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name-base demangled -k "regex:tc_gemm_kernel<.int.5" -s 2 -c 1 \
  -o gpurun_out/prof/lmhead_topk python tools/profile_steps.py > gpurun_out/prof/lmhead_topk.log 2>&1
