#!/bin/bash
for w in d116 t8; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fwd_$w.csv python tools/fwd_profile.py $w > gpurun_out/fwd_$w.log 2>&1
done
