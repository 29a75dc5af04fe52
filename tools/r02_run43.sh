#!/bin/bash
# round-2 GPU call 43: tcgen05 attention for prefill / long-row blocks (128-row tiles) - parity + A/B
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py -q -x > gpurun_out/r43_attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r43_attn_tests.log
grep -q "rc=0" gpurun_out/r43_attn_tests.log || exit 3
timeout 900 python -m pytest tests/test_llama_gpu.py tests/test_llama_bench_parity_gpu.py -q -x > gpurun_out/r43_llama_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r43_llama_tests.log
O=gpurun_out/r43_attn_rows.txt; : > $O
for t in 1 0; do
  echo "== FASER_ATTN_TC_ROWS=$t" >> $O
  FASER_ATTN_TC_ROWS=$t timeout 120 python tools/attn_bench.py 1,576,576 2,300,300 1,1000,1000 1,576,576,12,12,64 1,576,576,32,8,128 >> $O 2>&1
  FASER_ATTN_TC_ROWS=$t timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
  FASER_ATTN_TC_ROWS=$t timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-prefill-lane 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('nolane', round(d['value']), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
done
