#!/bin/bash
# round-2 GPU call 35: tcgen05 attention for GQA-packed rows - parity first, then timing
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention_gpu.py -q -x -k batch > gpurun_out/r35_attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r35_attn_tests.log
grep -q "rc=0" gpurun_out/r35_attn_tests.log || { timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_attention_gpu.py -q -x -k "batch and 32-4-64" > gpurun_out/r35_san.log 2>&1; exit 3; }
timeout 300 python -m pytest tests/test_attention_gpu.py -q > gpurun_out/r35_attn_all.log 2>&1; echo "rc=$?" >> gpurun_out/r35_attn_all.log
O=gpurun_out/r35_attn_tc.txt; : > $O
for t in 1 0; do
  echo "== FASER_ATTN_TC=$t" >> $O
  FASER_ATTN_TC=$t timeout 120 python tools/attn_bench.py 32,4,600 128,4,600 32,4,1000 32,4,600,32,8,128 >> $O 2>&1
done
