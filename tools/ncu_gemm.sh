mkdir -p gpurun_out
for shape in "3072 2048 116 0" "2048 8192 116 1" "4096 4096 8 1" "6144 4096 8 0"; do
  python tools/gemm_probe.py $shape 3 >> gpurun_out/probe.log 2>&1
  CARD_NO_CLUSTER=1 python tools/gemm_probe.py $shape 3 | sed 's/^/nocluster /' >> gpurun_out/probe.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/draft_qkv python tools/gemm_probe.py 3072 2048 116 0 3 > gpurun_out/ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/verify_o python tools/gemm_probe.py 4096 4096 8 1 3 > gpurun_out/ncu2.log 2>&1
