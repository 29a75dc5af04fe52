#!/bin/bash
# round-2 GPU call 47: tcgen05 ROW-block attention default: verify-row shapes A/B, llama tests, bench on/off
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_llama_gpu.py -q -x > gpurun_out/r47_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r47_tests.log
grep -q "rc=0" gpurun_out/r47_tests.log || exit 3
O=gpurun_out/r47_attn.txt; : > $O
for cfg in "FASER_ATTN_TC_ROWS=1" "FASER_ATTN_TC_ROWS=0"; do
  echo "== $cfg" >> $O
  env $cfg timeout 120 python tools/attn_bench.py 32,9,600 32,16,600 128,9,600 8,16,600 1,128,600 4,576,576 >> $O 2>&1
done
for cfg in "FASER_ATTN_TC_ROWS=1" "FASER_ATTN_TC_ROWS=0"; do
  env $cfg timeout 600 python bench.py > gpurun_out/r47_bench_$(echo $cfg | tr -d '=').json 2> gpurun_out/r47_bench_$(echo $cfg | tr -d '=').err
done
