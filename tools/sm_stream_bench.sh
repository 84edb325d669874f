#!/bin/bash
# per-SM streaming: TMA bulk vs LDG vs both (tools/sm_stream_bench.cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smbench tools/sm_stream_bench.cu || exit 1
for c in 16 64 128 148; do for m in 0 1 2; do timeout 60 /tmp/smbench $c $m 4; done; done
