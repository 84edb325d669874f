#!/bin/bash
# A/B two builds (abtest/old.so, abtest/new.so) on one box: bench.py serial (2 rounds) + microbench d116 topk
mkdir -p gpurun_out
for r in 1 2; do for v in old new; do
  cp abtest/$v.so paper_2508_04462_b200/libcard_b200.so
  echo "== $v round $r"; timeout 800 python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['speedup_vs_ar'], d['mean_acceptance_length'], d['lossless_vs_ar'])"
  timeout 300 python tools/microbench.py d116 | grep -E "topk|graph replay"
done; done
cp abtest/new.so paper_2508_04462_b200/libcard_b200.so
