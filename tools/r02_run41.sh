#!/bin/bash
# round-2 GPU call 41: recovery on prune (exempt_rule 2): parity, then EE+recovery vs VSD benches
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_llama_gpu.py -q -x -k "recovery or early_exit or lossless" > gpurun_out/r41_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r41_tests.log
grep -q "rc=0" gpurun_out/r41_tests.log || exit 3
O=gpurun_out/r41_recovery.txt; : > $O
for B in 32 128 256; do for m in "vsd" "vsd_ee --gate-layer 2 --recovery" "vsd_ee --gate-layer 2"; do
echo "== B=$B $m" >> $O
timeout 600 python bench.py --steps 40 --warmup 5 --batch $B --mode $m --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), round(d['p50_tpot_ms'],3), round(d['acceptance'],3), round(d['layer_work_per_drafted_token'],2), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
done; done
