#!/bin/bash
# round-2 GPU call 49: tcgen05 GROUP attention by default above 32 packed rows: tests, bench A/B
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_llama_gpu.py -q -x > gpurun_out/r49_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r49_tests.log
grep -q "rc=0" gpurun_out/r49_tests.log || exit 3
for cfg in "FASER_ATTN_TC=0" "FASER_ATTN_X=1" "FASER_ATTN_TC=0" "FASER_ATTN_X=1"; do
  env $cfg timeout 600 python bench.py >> gpurun_out/r49_bench_$(echo $cfg | tr -d '=').json 2>> gpurun_out/r49_bench.err
done
