#!/bin/bash
# round-2 GPU call 84: config 4 in-stream A/B of the sweep-driven planner (FASER_GEMM_PLAN=table) vs rules+legacy
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/r84_ab.jsonl
for rep in 1 2; do for cfg in "FASER_GEMM_PLAN=default" "FASER_GEMM_PLAN=table"; do
  echo "{\"cfg\": \"$cfg\"}" >> gpurun_out/r84_ab.jsonl
  env $cfg timeout 1200 python bench.py --workload cfg4 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r84_ab.jsonl
done; done
