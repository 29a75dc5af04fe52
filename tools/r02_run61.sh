#!/bin/bash
# round-2 GPU call 61: split-KV only for long contexts: attention tests (+ long shape), small-batch A/B, B=8 bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_llama_gpu.py -q -x > gpurun_out/r61_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r61_tests.log
grep -q "rc=0" gpurun_out/r61_tests.log || exit 3
O=gpurun_out/r61_attn.txt; : > $O
for r in 0 1; do
  echo "== RAGGED=$r (new default)" >> $O
  ATTN_BENCH_RAGGED=$r timeout 120 python tools/attn_bench.py 1,4,600 1,4,2000 4,4,600 8,4,600 16,4,600 1,1,600 8,1,600 1,5,600,12,12,64 8,1,600,12,12,64 >> $O 2>&1
done
for b in 1 8; do
  timeout 600 python bench.py --batch $b --steps 40 --warmup 6 --no-sweep --no-cpu-baseline >> gpurun_out/r61_bench_small.jsonl 2>> gpurun_out/r61_bench.err
done
