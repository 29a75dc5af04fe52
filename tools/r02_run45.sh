#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
FASER_ATTN_TC=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_tc -c 1 -o gpurun_out/r45_tc python tools/attn_bench.py 32,4,600 > gpurun_out/r45_ncu.log 2>&1
