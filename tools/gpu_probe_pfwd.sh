# persistent forward: agreement + replay time, timeline, tree parity (gpurun_out/pf/)
mkdir -p gpurun_out/pf
O=gpurun_out/pf
timeout 300 python tools/pfwd_probe.py > $O/probe.log 2>&1; echo "rc=$?" >> $O/probe.log
timeout 300 python tools/pfwd_trace.py > $O/trace.log 2>&1; echo "rc=$?" >> $O/trace.log
timeout 300 python -m pytest tests/test_gpu_parity_full.py -q -x -k tree -s > $O/tree.log 2>&1; echo "rc=$?" >> $O/tree.log
