#!/bin/bash
# round-2 GPU call 37: attention tests incl. the opt-in tcgen05 kernel; A/B timing
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py -q > gpurun_out/r37_attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r37_attn_tests.log
O=gpurun_out/r37_attn_tc.txt; : > $O
for t in 1 0; do
  echo "== FASER_ATTN_TC=$t" >> $O
  FASER_ATTN_TC=$t timeout 120 python tools/attn_bench.py 32,4,600 128,4,600 32,4,1000 32,4,600,32,8,128 >> $O 2>&1
done
