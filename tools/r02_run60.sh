#!/bin/bash
# round-2 GPU call 60: split-KV on/off at small batches (FASER_ATTN_CTAS=1 disables the split)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r60_attn_nosplit.txt; : > $O
for r in 0 1; do for c in 1 148; do
  echo "== RAGGED=$r FASER_ATTN_CTAS=$c" >> $O
  ATTN_BENCH_RAGGED=$r FASER_ATTN_CTAS=$c timeout 120 python tools/attn_bench.py 1,4,600 1,4,2000 4,4,600 8,4,600 16,4,600 1,1,600 8,1,600 1,5,600,12,12,64 8,1,600,12,12,64 >> $O 2>&1
done; done
