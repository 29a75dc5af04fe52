#!/bin/bash
# round-2 GPU call 63: ncu source-level of the mma.sync GROUP attention (32 x 4 rows, ctx 1000)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -c 1 -o gpurun_out/r63_mma python tools/attn_bench.py 32,4,1000 > gpurun_out/r63_ncu.log 2>&1
