#!/bin/bash
# A/B two builds of libcard_b200.so on one box: abtest/old.so vs abtest/new.so (forward microbench, 2 rounds)
mkdir -p gpurun_out
for r in 1 2; do for v in old new; do
  cp abtest/$v.so paper_2508_04462_b200/libcard_b200.so
  echo "== $v round $r"; timeout 300 python tools/microbench.py t1 t8 d116 | grep "graph replay"
done; done
cp abtest/new.so paper_2508_04462_b200/libcard_b200.so
