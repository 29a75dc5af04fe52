#!/bin/bash
# round-2 GPU call 73: toy config-2 bench (no profiling), 3 repeats + reference arm
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/r73_toy.jsonl
for i in 1 2 3; do timeout 300 python bench.py --workload toy --steps 200 --warmup 20 >> gpurun_out/r73_toy.jsonl 2>> gpurun_out/r73_toy.err; done
timeout 300 python bench.py --workload toy --impl reference --steps 200 --warmup 20 > gpurun_out/r73_toy_ref.json 2>> gpurun_out/r73_toy.err
