#!/bin/bash
# round-2 GPU call 11: compute-sanitizer (racecheck / synccheck / memcheck) on the GEMM, attention,
# FULL-mode lanes and early-exit tests; TP (bf16 all-reduce) tests; then the whole GPU suite
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r11_sanitizer.txt; : > $O
san() { tool=$1; shift; echo "=== compute-sanitizer --tool $tool :: $*" >> $O;
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python -m pytest -q -x "$@" > /tmp/san.log 2>&1; rc=$?
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|error" /tmp/san.log | tail -4 >> $O; echo "rc=$rc" >> $O; }
san racecheck "tests/test_gemm_gpu.py::test_gemm_matches_fp32" -k "2560 and 128"
san synccheck "tests/test_gemm_gpu.py::test_gemm_matches_fp32" -k "2560 and 128"
san racecheck tests/test_attention_gpu.py -k "verify or decode"
san synccheck tests/test_attention_gpu.py -k "verify"
san memcheck tests/test_lanes_gpu.py -k "early_exit_inside_chunks"
san synccheck tests/test_lanes_gpu.py -k "early_exit_inside_chunks"
san memcheck tests/test_llama_gpu.py -k "early_exit_decisions and tiny-"
timeout 900 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r11_gpu_tests.log 2>&1; echo "suite rc=$?" >> gpurun_out/r11_gpu_tests.log
