#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r27_pfdebug.txt; : > $O
for B in 128 256; do
echo "== B=$B" >> $O
FASER_PF_DEBUG=1 timeout 400 python bench.py --steps 20 --warmup 5 --batch $B --no-sweep --no-cpu-baseline 2>>$O | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), d['wall_s_timed'], {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
done
