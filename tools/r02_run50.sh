#!/bin/bash
# round-2 GPU call 50: which attention kernel the bench's verify forwards dispatch
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
FASER_ATTN_DEBUG=400 timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r50_bench.json 2> gpurun_out/r50_dbg.txt
