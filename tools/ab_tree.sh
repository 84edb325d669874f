#!/bin/bash
# Same-box A/B of two whole trees (abtest/old = an earlier commit, built; . = current):
# draft / target step graph times (tools/step_times.py), two rounds
mkdir -p gpurun_out/ab
for r in 1 2; do
  for v in old new; do
    d=.; [ $v = old ] && d=abtest/old
    echo "== $v round $r"
    (cd $d && SHARP=1e6 NEW=128 timeout 300 python tools/step_times.py 2>&1 | grep -E "steps|committed")
  done
done
