#!/bin/bash
# round-2 GPU call 87: warp-per-page decode attention for the MHA draft: tests, A/B, bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_llama_gpu.py tests/test_llama_bench_parity_gpu.py -q -x > gpurun_out/r87_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r87_tests.log
grep -q "rc=0" gpurun_out/r87_tests.log || { timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_attention_gpu.py -q -x -k "decode and 12-12" > gpurun_out/r87_san.log 2>&1; exit 3; }
O=gpurun_out/r87_attn.txt; : > $O
for r in 0 1; do for d in 1 0; do
  echo "== RAGGED=$r FASER_ATTN_DECODE=$d" >> $O
  ATTN_BENCH_RAGGED=$r FASER_ATTN_DECODE=$d timeout 120 python tools/attn_bench.py 32,1,600,12,12,64 128,1,600,12,12,64 8,1,600,12,12,64 32,1,1500,12,12,64 >> $O 2>&1
done; done
for d in 1 0 1 0; do
  echo "{\"FASER_ATTN_DECODE\": $d}" >> gpurun_out/r87_bench.jsonl
  FASER_ATTN_DECODE=$d timeout 600 python bench.py --steps 30 --warmup 6 --no-sweep --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r87_bench.jsonl
done
