#!/bin/bash
# Round pass on one B200: GPU tests, smoke, the bench line, agreement-knob sweep, ncu launch list
mkdir -p gpurun_out/round
O=gpurun_out/round
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_serial.log 2>&1
NEW=256 timeout 900 python tools/bias_sweep.py > $O/bias_sweep.log 2>&1
mkdir -p gpurun_out/prof
NEW=32 SHARP=1e6 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches_card.csv python tools/profile_steps.py > gpurun_out/prof/launches_card.log 2>&1
echo done > $O/done
