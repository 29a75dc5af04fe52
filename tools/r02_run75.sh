#!/bin/bash
# round-2 GPU call 75: pair split only when each CTA keeps its own SM: tests, sanitizer on the pair shape, small-batch bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_llama_gpu.py -q -x > gpurun_out/r75_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r75_tests.log
grep -q "rc=0" gpurun_out/r75_tests.log || exit 3
for tool in racecheck synccheck memcheck; do
  echo "== $tool" >> gpurun_out/r75_san.txt
  timeout 600 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_attention_gpu.py -q -x -k "pair" >> gpurun_out/r75_san.txt 2>&1; echo "rc=$?" >> gpurun_out/r75_san.txt
done
O=gpurun_out/r75_attn.txt; : > $O
ATTN_BENCH_RAGGED=1 timeout 120 python tools/attn_bench.py 32,4,600 16,4,600 8,4,600 4,4,600 >> $O 2>&1
for b in 8 16; do timeout 600 python bench.py --batch $b --steps 40 --warmup 6 --no-sweep --no-cpu-baseline >> gpurun_out/r75_bench.jsonl 2>> gpurun_out/r75_bench.err; done
