#!/bin/bash
# round-2 GPU call 48: GROUP-row attention occupancy: KV-split CTA target sweep, uniform and ragged contexts
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r48_attn_split.txt; : > $O
for r in 0 1; do for c in 148 296 444 592 888 1184; do
  echo "== RAGGED=$r FASER_ATTN_CTAS=$c" >> $O
  ATTN_BENCH_RAGGED=$r FASER_ATTN_CTAS=$c timeout 120 python tools/attn_bench.py 32,5,600 32,5,1000 128,5,600 32,5,600,32,8,128 8,5,600 >> $O 2>&1
done; done
echo "== RAGGED=1 FASER_ATTN_TC=1" >> $O
ATTN_BENCH_RAGGED=1 FASER_ATTN_TC=1 timeout 120 python tools/attn_bench.py 32,5,600 32,5,1000 128,5,600 32,5,600,32,8,128 8,5,600 >> $O 2>&1
