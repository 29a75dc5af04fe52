#!/bin/bash
# round-2 GPU call 66: toy step host anatomy (FASER_TOY_PROF)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
FASER_TOY_PROF=1 timeout 300 python bench.py --workload toy --steps 200 --warmup 20 > gpurun_out/r66_toy.json 2> gpurun_out/r66_toy.err
