#!/bin/bash
# round-2 GPU call 40: split-K reduce with batched DSMEM loads + split cluster arrive/wait
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/r40_gemm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r40_gemm_tests.log
grep -q "rc=0" gpurun_out/r40_gemm_tests.log || exit 3
O=gpurun_out/r40_chain.jsonl; : > $O
for r in 128 32 256; do echo "# rows $r" >> $O; timeout 120 python tools/layer_chain.py --rows $r --trace >> $O 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(json.dumps({'bench':round(d['value']), 'ms':round(d['ms_per_step'],3), 'dev':{k:round(v,3) for k,v in d['device_ms_per_step'].items()}, 'instream':d['roofline'].get('instream')}))" >> $O
