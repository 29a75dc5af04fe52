#!/bin/bash
# round-2 GPU call 28: cap on prefill batches in flight on the lane (launch-queue back-pressure)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_llama_gpu.py -q -x -k "prefill_lane or lossless" > gpurun_out/r28_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r28_tests.log
O=gpurun_out/r28_inflight.txt; : > $O
for B in 128 32 256; do for c in 1 2 4 16; do
echo "== B=$B inflight=$c" >> $O
FASER_PF_DEBUG=1 FASER_PF_INFLIGHT=$c timeout 400 python bench.py --steps 20 --warmup 5 --batch $B --no-sweep --no-cpu-baseline 2>>$O | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), round(d['p50_tpot_ms'],3), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
done; done
