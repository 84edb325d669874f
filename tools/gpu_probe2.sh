#!/bin/bash
mkdir -p gpurun_out/p2
O=gpurun_out/p2
timeout 300 python tools/attn_tree_probe.py 1000 10 > $O/attn.log 2>&1; echo "rc=$?" >> $O/attn.log
timeout 300 python tools/attn_tree_probe.py 600 14 >> $O/attn.log 2>&1; echo "rc=$?" >> $O/attn.log
timeout 300 python tools/pfwd_trace.py > $O/pfwd_trace.log 2>&1; echo "rc=$?" >> $O/pfwd_trace.log
