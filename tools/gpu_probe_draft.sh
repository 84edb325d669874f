#!/bin/bash
# Draft-step breakdown: per-graph step times, persistent-forward timeline, ncu launch list (gpurun_out/dp/)
mkdir -p gpurun_out/dp
O=gpurun_out/dp
SHARP=1e6 NEW=128 timeout 300 python tools/step_times.py > $O/step_times.log 2>&1; echo "rc=$?" >> $O/step_times.log
timeout 300 python tools/pfwd_trace.py > $O/pfwd_trace.log 2>&1; echo "rc=$?" >> $O/pfwd_trace.log
NEW=32 SHARP=1e6 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_card.csv python tools/profile_steps.py > $O/launches_card.log 2>&1; echo "rc=$?" >> $O/launches_card.log
