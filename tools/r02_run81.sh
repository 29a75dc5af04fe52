#!/bin/bash
# round-2 GPU call 81: in-stream A/B of the sweep-driven planner on the configs' own shapes (bench B=32 and B=128)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/r81_ab.jsonl
for rep in 1 2; do for cfg in "FASER_GEMM_PLAN=default" "FASER_GEMM_PLAN=table"; do for b in 32 128; do
  echo "{\"cfg\": \"$cfg\", \"batch\": $b}" >> gpurun_out/r81_ab.jsonl
  env $cfg timeout 600 python bench.py --batch $b --steps 30 --warmup 6 --no-sweep --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r81_ab.jsonl
done; done; done
