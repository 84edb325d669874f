mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:ILi5ELb0 -c 1 -s 1 -o gpurun_out/topk_head python tools/topk_probe_one.py > gpurun_out/ncu_topk.log 2>&1
