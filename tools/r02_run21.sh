#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for a in "--no-prefill-lane" ""; do
timeout 900 python bench.py --workload cfg4 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline $a 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$a', round(d['value']), round(d['ms_per_step'],3), round(d['p50_tpot_ms'],3), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> gpurun_out/r21_cfg4.txt
done
