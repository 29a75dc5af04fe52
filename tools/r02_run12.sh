#!/bin/bash
# round-2 GPU call 12: step breakdown (admission/prefill, draft, verify) + in-stream class shares
# via FASER_SKIP (results garbage, timing only), GEMM sanitizer
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r12_breakdown.txt; : > $O
b() { echo "== $*" >> $O; env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['device_ms_per_step'].items()})" >> $O 2>&1; }
b FASER_SKIP=0
b FASER_SKIP=1
b FASER_SKIP=30
b FASER_SKIP=33
b FASER_SKIP=62
b FASER_SKIP=0
S=gpurun_out/r12_sanitizer.txt; : > $S
san() { tool=$1; shift; echo "=== compute-sanitizer --tool $tool :: $*" >> $S;
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python -m pytest -q -x "$@" > /tmp/san.log 2>&1; rc=$?
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rror" /tmp/san.log | tail -4 >> $S; echo "rc=$rc" >> $S; }
san racecheck tests/test_gemm_gpu.py -k "test_gemm_matches_fp32 and 2560-20-2048"
san synccheck tests/test_gemm_gpu.py -k "test_gemm_matches_fp32 and 2560-20-2048"
san memcheck tests/test_gemm_gpu.py -k "test_gemm_matches_fp32 and (2560-20-2048 or 11264-160-2048)"
