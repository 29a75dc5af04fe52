#!/bin/bash
# round-2 GPU call 51: tcgen05 attention with 8 softmax warps (key halves)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py -q -x > gpurun_out/r51_attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r51_attn_tests.log
grep -q "rc=0" gpurun_out/r51_attn_tests.log || { timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_attention_gpu.py -q -x -k "prefill and 32-4-64" > gpurun_out/r51_san.log 2>&1; exit 3; }
O=gpurun_out/r51_attn.txt; : > $O
for cfg in "FASER_ATTN_TC=1 FASER_ATTN_TC_ROWS=1" "FASER_ATTN_TC=0 FASER_ATTN_TC_ROWS=0" "ATTN_BENCH_RAGGED=1 FASER_ATTN_TC=1" "ATTN_BENCH_RAGGED=1 FASER_ATTN_TC=0"; do
  echo "== $cfg" >> $O
  env $cfg timeout 120 python tools/attn_bench.py 32,4,600 128,4,600 32,5,600 128,5,600 32,4,600,32,8,128 1,576,576 1,1000,1000 1,576,576,32,8,128 32,16,600 >> $O 2>&1
done
