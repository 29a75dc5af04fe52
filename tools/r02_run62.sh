#!/bin/bash
# round-2 GPU call 62: mma.sync attention pipeline depth (compile-time variants 3/4/6/8 stages), hd 64
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r62_attn_stages.txt; : > $O
for v in base attn_st4 attn_st6 attn_st8; do
  lib=""; [ "$v" != base ] && lib="$PWD/build/variants/$v.so"
  for r in 0 1; do
    echo "== $v RAGGED=$r" >> $O
    FASER_LIB=$lib ATTN_BENCH_RAGGED=$r timeout 120 python tools/attn_bench.py 32,1,600,12,12,64 32,4,600 32,4,1000 8,4,600 128,4,600 1,4,2000 >> $O 2>&1
  done
done
