#!/bin/bash
# round-2 GPU call 29: lane in-flight cap at longer windows (60 steps)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r29_inflight.txt; : > $O
for B in 32 128; do for c in 2 4 16; do
echo "== B=$B inflight=$c" >> $O
FASER_PF_INFLIGHT=$c timeout 600 python bench.py --steps 60 --warmup 5 --batch $B --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), round(d['p50_tpot_ms'],3), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
done; done
echo "== B=32 no lane" >> $O
timeout 600 python bench.py --steps 60 --warmup 5 --batch 32 --no-sweep --no-cpu-baseline --no-prefill-lane 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), round(d['p50_tpot_ms'],3), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
