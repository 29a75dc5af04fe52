#!/bin/bash
# round-2 GPU call 14: TMA box-size probe (L2-resident and HBM) at GEMM-like in-flight bytes
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r14_tma_box.jsonl; : > $O
for mode in 2 0; do
for cfg in "100 24 32 1" "100 6 128 1" "100 12 32 4" "100 3 128 4" "100 48 32 1" "100 12 128 1" "148 24 32 1" "148 6 128 1" "100 6 32 4" "100 24 32 4"; do
  set -- $cfg
  for v in 0 3; do timeout 60 ./tools/tma_probe $mode $1 $2 $3 $4 $v >> $O 2>&1; done
done; done
