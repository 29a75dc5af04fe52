#!/bin/bash
# round-2 GPU call 17: admission-prefill lane (side stream) - losslessness + bench A/B
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_llama_gpu.py -q -x tests/test_lanes_gpu.py > gpurun_out/r17_lane_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r17_lane_tests.log
grep -q "rc=0" gpurun_out/r17_lane_tests.log || exit 3
O=gpurun_out/r17_lane_bench.txt; : > $O
for a in "" "--no-prefill-lane" "" "--no-prefill-lane" "--batch 128" "--batch 128 --no-prefill-lane"; do
echo "== $a" >> $O
timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline $a 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), round(d['p50_tpot_ms'],3), d['e2e']['value'], {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1
done
