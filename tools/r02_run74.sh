#!/bin/bash
# round-2 GPU call 74: cluster-pair split-KV for GROUP attention (DSMEM merge): tests + A/B
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py -q -x > gpurun_out/r74_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r74_tests.log
grep -q "rc=0" gpurun_out/r74_tests.log || { timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_attention_gpu.py -q -x -k "verify and 32-4-64" > gpurun_out/r74_san.log 2>&1; exit 3; }
O=gpurun_out/r74_attn.txt; : > $O
for r in 0 1; do for p in 0 6 4; do
  echo "== RAGGED=$r FASER_ATTN_PAIR=$p" >> $O
  ATTN_BENCH_RAGGED=$r FASER_ATTN_PAIR=$p timeout 120 python tools/attn_bench.py 32,4,600 32,4,1000 32,4,300 16,4,600 8,4,600 36,4,600 32,4,600,32,8,128 32,1,600,12,12,64 >> $O 2>&1
done; done
