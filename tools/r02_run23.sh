#!/bin/bash
# round-2 GPU call 23: attention page loads via TMA by default (hd 64 and 128, one box layout)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_llama_gpu.py tests/test_llama_bench_parity_gpu.py tests/test_tp_gpu.py -q -x > gpurun_out/r23_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r23_tests.log
grep -q "rc=0" gpurun_out/r23_tests.log || exit 3
O=gpurun_out/r23_attn_tma.txt; : > $O
for t in 1 0; do
  echo "== FASER_ATTN_TMA=$t" >> $O
  FASER_ATTN_TMA=$t timeout 120 python tools/attn_bench.py 32,4,600 32,1,600,12,12,64 128,4,600 32,4,600,32,8,128 32,1,600,32,8,64 >> $O 2>&1
  FASER_ATTN_TMA=$t timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['device_ms_per_step'].items()}, {k:round(v['avg_us'],2) for k,v in d['kernels'].items()})" >> $O 2>&1
done
