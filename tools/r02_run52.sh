#!/bin/bash
# round-2 GPU call 52: ncu of the 8-softmax-warp tcgen05 attention (32x4 rows, ctx 600)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
FASER_ATTN_TC=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_tc -c 1 -o gpurun_out/r52_tc python tools/attn_bench.py 32,4,600 > gpurun_out/r52_ncu.log 2>&1
