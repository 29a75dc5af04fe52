#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
FASER_ATTN_TC_TRACE=1 timeout 120 python tools/attn_bench.py 32,4,600 > gpurun_out/r36_trace.txt 2>&1
