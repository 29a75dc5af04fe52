#!/bin/bash
# round-2 GPU call 83: config 4 (8B target) bench line at HEAD
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python bench.py --workload cfg4 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline > gpurun_out/r83_cfg4.json 2> gpurun_out/r83_cfg4.err
