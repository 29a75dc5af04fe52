#!/bin/bash
# round-2 GPU call 59: bench line with mean TPOT / accepted-draft tok/s; full batch sweep points 2,4,16,64; attention KV-split at B=32 rows=4
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline > gpurun_out/r59_bench.json 2> gpurun_out/r59_bench.err
: > gpurun_out/r59_sweep.jsonl
for b in 2 4 16 64; do
  timeout 600 python bench.py --batch $b --steps 40 --warmup 6 --no-sweep --no-cpu-baseline >> gpurun_out/r59_sweep.jsonl 2>> gpurun_out/r59_bench.err
done
O=gpurun_out/r59_attn_split.txt; : > $O
for c in 148 256 384 512; do
  echo "== FASER_ATTN_CTAS=$c" >> $O
  ATTN_BENCH_RAGGED=1 FASER_ATTN_CTAS=$c timeout 120 python tools/attn_bench.py 32,4,600 32,4,1000 16,4,600 >> $O 2>&1
done
