#!/bin/bash
# round-2 GPU call 54: attention TMA issue lanes rotating with the page/step (per-thread box serialisation)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py -q -x > gpurun_out/r54_attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r54_attn_tests.log
grep -q "rc=0" gpurun_out/r54_attn_tests.log || exit 3
O=gpurun_out/r54_attn.txt; : > $O
for cfg in "FASER_ATTN_TC=1" "FASER_ATTN_TC=0" "ATTN_BENCH_RAGGED=1 FASER_ATTN_TC=1" "ATTN_BENCH_RAGGED=1 FASER_ATTN_TC=0"; do
  echo "== $cfg" >> $O
  env $cfg timeout 120 python tools/attn_bench.py 32,4,64 32,4,256 32,4,600 32,4,1024 32,4,2048 128,4,600 32,5,600 8,4,600 1,4,600 32,4,600,32,8,128 1,576,576 >> $O 2>&1
done
