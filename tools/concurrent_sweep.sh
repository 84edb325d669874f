#!/bin/bash
mkdir -p gpurun_out/cc
for x in "concurrent events --draft-per-gemm" "concurrent events" "serial_sim events --draft-per-gemm" "concurrent mailbox --draft-per-gemm"; do
  set -- $x
  echo "== $x"
  timeout 600 python bench.py --mode $1 $( [ $1 = concurrent ] && echo --exchange $2 ) $3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/cc/b.log 2>&1; echo "exit $?"
  tail -1 gpurun_out/cc/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['speedup_vs_ar'], d['mean_acceptance_length'], d['lossless_vs_ar'])" 2>&1 | tail -1
done
