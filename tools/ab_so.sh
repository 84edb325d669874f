#!/bin/bash
# Same-box A/B of library builds abtest/<name>.so (same Python tree): persistent-forward
# timeline and draft/target step times.  Usage: ab_so.sh name1 name2 ...
for r in 1 2; do for v in "$@"; do
  cp abtest/$v.so paper_2508_04462_b200/libcard_b200.so
  echo "== $v round $r"
  timeout 300 python tools/pfwd_trace.py 2>&1 | grep -E "L 1\.gu|all pfwd"
  SHARP=1e6 NEW=128 timeout 300 python tools/step_times.py 2>&1 | grep -E "^draft steps|^target steps"
done; done
cp abtest/new.so paper_2508_04462_b200/libcard_b200.so
