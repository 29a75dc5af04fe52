#!/bin/bash
# round-2 GPU call 10: fused exit-test estimator (no T x V logits): parity + vsd_ee bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_llama_gpu.py tests/test_lanes_gpu.py -q -x > gpurun_out/r10_ee_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r10_ee_tests.log
grep -q "rc=0" gpurun_out/r10_ee_tests.log || exit 3
timeout 600 python -m pytest tests/test_llama_bench_parity_gpu.py -q -x > gpurun_out/r10_bp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r10_bp_tests.log
: > gpurun_out/r10_ee_bench.txt
for B in 32 128; do for m in "vsd_ee --gate-layer 2" "vsd_ee --gate-layer 8" "vsd"; do
echo "== B=$B $m" >> gpurun_out/r10_ee_bench.txt
timeout 300 python bench.py --steps 30 --warmup 5 --batch $B --mode $m --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), d['ms_per_step'], d['acceptance'], d['device_ms_per_step'], {k:round(v['avg_us'],2) for k,v in d['kernels'].items()})" >> gpurun_out/r10_ee_bench.txt 2>&1
done; done
