#!/bin/bash
# round-2 GPU call 85: full plan sweep of the config-4 draft shapes at 32 rows (+ the engine's current plans)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python tools/plan_fit_sweep.py 3072,32,2048 2048,32,2048 16384,32,2048 2048,32,8192 128256,32,2048 > gpurun_out/r85_c4d.jsonl 2> gpurun_out/r85_c4d.err
