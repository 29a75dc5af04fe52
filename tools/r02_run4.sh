#!/bin/bash
# round-2 GPU call 4: lane profile (SM-share latency samples + interference), FULL-mode bench lines
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python tools/lane_profile.py > gpurun_out/r4_lane_profile.log 2>&1; echo "rc=$?" >> gpurun_out/r4_lane_profile.log
for m in "vsd" "full --chunk 2"; do
  timeout 600 python bench.py --steps 40 --warmup 5 --batch 32 --k 4 --mode $m --no-cpu-baseline --no-sweep >> gpurun_out/r4_modes.jsonl 2>> gpurun_out/r4_modes.err
done
