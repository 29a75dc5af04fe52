#!/bin/bash
# round-2 GPU call 31: short prefill CTAs on the lane (FASER_PF_TILES=small) vs the prefill plans (60 steps)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r31_pftiles.txt; : > $O
for B in 32 128; do for t in small big; do
echo "== B=$B tiles=$t" >> $O
FASER_PF_TILES=$t timeout 600 python bench.py --steps 60 --warmup 5 --batch $B --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), round(d['p50_tpot_ms'],3), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
done; done
