#!/bin/bash
# round-2 GPU call 58: compute-sanitizer on the tcgen05 attention (ROW blocks + GROUP > 32 rows, default dispatch)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r58_san.txt; : > $O
for tool in memcheck racecheck synccheck; do
  echo "=== compute-sanitizer --tool $tool :: tests/test_attention_gpu.py -k (prefill or batch or ragged) and (32-4-64 or 32-8-128)" >> $O
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_attention_gpu.py -q -x -k "(prefill or batch or ragged) and (32-4-64 or 32-8-128) and matches_fp32" >> $O 2>&1
  echo "rc=$?" >> $O
done
