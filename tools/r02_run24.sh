#!/bin/bash
# round-2 GPU call 25: prefill-lane blob ring 4 -> 16 (no host wait on ring wrap at large B)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r25_ring.txt; : > $O
for B in 128 256 32; do for a in "" "--no-prefill-lane"; do
echo "== B=$B $a" >> $O
timeout 400 python bench.py --steps 20 --warmup 5 --batch $B --no-sweep --no-cpu-baseline $a 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), round(d['p50_tpot_ms'],3), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
done; done
