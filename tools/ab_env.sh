#!/bin/bash
# A/B an environment knob on one box: bench.py serial without vs with "$@" (2 rounds)
mkdir -p gpurun_out
for r in 1 2; do for v in base knob; do
  if [ $v = knob ]; then E="$*"; else E=""; fi
  echo "== $v [$E] round $r"
  env $E timeout 800 python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['speedup_vs_ar'], d['ar_tokens_per_s'], d['mean_acceptance_length'], d['lossless_vs_ar'])"
done; done
