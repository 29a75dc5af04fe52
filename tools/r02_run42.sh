#!/bin/bash
# round-2 GPU call 42: ablation ladder on the steady-state bench (config 3): VSD -> AD -> AD+EE -> FULL, with recovery
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r42_modes.txt; : > $O
for B in 32 128; do for m in "vsd" "ad" "ee" "ee --recovery" "vsd_ee --recovery" "full"; do
echo "== B=$B $m" >> $O
timeout 600 python bench.py --steps 40 --warmup 5 --batch $B --mode $m --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), round(d['p50_tpot_ms'],3), round(d['acceptance'],3), round(d['layer_work_per_drafted_token'],2), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
done; done
