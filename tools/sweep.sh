#!/bin/bash
# Batch sweep of the headline metric (config 3, 1 GPU): one bench.py JSON line per batch size.
out=${1:-gpurun_out/sweep.jsonl}
: > "$out"
for b in 1 2 4 8 16 32 64 128 256; do
  timeout 400 python bench.py --batch $b --steps ${STEPS:-40} --warmup 6 --no-cpu-baseline --mode ${MODE:-vsd} 2>/dev/null | tail -1 >> "$out"
done
