#!/bin/bash
# launch list of one CARD request + AR (requests only) -> gpurun_out/prof/launches_card.csv
mkdir -p gpurun_out/prof
NEW=32 SHARP=${SHARP:-1e6} timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches_card.csv python tools/profile_steps.py > gpurun_out/prof/launches_card.log 2>&1
