#!/bin/bash
# round-2 GPU call 98: config 5 (70B-shape target, 141 GB bf16) instantiated on ONE B200 at TP=1 (fits 180 GB HBM): bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
(while true; do nvidia-smi --query-gpu=memory.used,memory.total,clocks.sm --format=csv,noheader >> gpurun_out/r98_mem.txt; sleep 5; done) &
MON=$!
timeout 1200 python bench.py --workload cfg5 --batch 8 --steps 8 --warmup 3 > gpurun_out/r98_cfg5_tp1.json 2> gpurun_out/r98_cfg5_tp1.err; echo "rc=$?" >> gpurun_out/r98_cfg5_tp1.err
kill $MON
