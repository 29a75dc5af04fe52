#!/bin/bash
# round-2 GPU call 15: one activation TMA box per stage (64/128/256-row boxes) vs 32-row boxes
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/r15_gemm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r15_gemm_tests.log
grep -q "rc=0" gpurun_out/r15_gemm_tests.log || exit 3
O=gpurun_out/r15_xbox.jsonl; : > $O
for xb in 256 32; do
  echo "# XBOX=$xb" >> $O
  FASER_XBOX=$xb timeout 120 python tools/gemm_bench.py 2560,576,2048 11264,576,2048 2048,576,5632 2048,576,2048 2560,128,2048 11264,128,2048 11264,1024,2048 >> $O 2>&1
  for r in 128 512; do FASER_XBOX=$xb timeout 120 python tools/layer_chain.py --rows $r >> $O 2>&1; done
  FASER_XBOX=$xb timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(json.dumps({'bench':round(d['value']), 'ms':round(d['ms_per_step'],3), 'dev':{k:round(v,3) for k,v in d['device_ms_per_step'].items()}}))" >> $O
done
