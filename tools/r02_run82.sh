#!/bin/bash
# round-2 GPU call 82: prefill forwards on the sweep-driven planner (FASER_PREFILL_PLAN=table) vs rules, B=32 / 128 / 256
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/r82_ab.jsonl
for rep in 1 2; do for cfg in "FASER_PREFILL_PLAN=rules" "FASER_PREFILL_PLAN=table"; do for b in 32 128 256; do
  echo "{\"cfg\": \"$cfg\", \"batch\": $b}" >> gpurun_out/r82_ab.jsonl
  env $cfg timeout 600 python bench.py --batch $b --steps 30 --warmup 6 --no-sweep --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r82_ab.jsonl
done; done; done
