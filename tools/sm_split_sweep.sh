#!/bin/bash
# mode=concurrent on one B200 with the SMs split between draft and target (card_green)
mkdir -p gpurun_out/sms
for x in "0 events" "48 events" "64 events" "80 events" "64 mailbox"; do
  set -- $x
  echo "== draft_sms=$1 exchange=$2"
  timeout 600 python bench.py --mode concurrent --draft-sms $1 --exchange $2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/sms/b_$1_$2.log 2>&1; echo "exit $?"; tail -1 gpurun_out/sms/b_$1_$2.log | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['speedup_vs_ar'], d['mean_acceptance_length'], d['lossless_vs_ar'])" 2>&1 | tail -2
done
