#!/bin/bash
# round-2 GPU call 68: ncu source-level of the fused toy round kernel
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:draft_verify -s 40 -c 1 -o gpurun_out/r68_toy python bench.py --workload toy --steps 60 --warmup 5 > gpurun_out/r68_ncu.log 2>&1
