#!/bin/bash
# round-2 GPU call 80: sweep-driven GEMM planner: full GPU suite + out-of-sample sweep (Phi-3-mini / Yi-6B-like shapes)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r80_gpu_tests.log 2>&1; echo "suite rc=$?" >> gpurun_out/r80_gpu_tests.log
timeout 2400 python tools/plan_fit_sweep.py 9216,32,3072 3072,32,3072 16384,32,3072 3072,32,8192 5120,32,4096 22016,32,4096 4096,32,11008 9216,128,3072 3072,128,3072 16384,128,3072 3072,128,8192 5120,128,4096 22016,128,4096 4096,128,11008 9216,512,3072 3072,512,3072 16384,512,3072 3072,512,8192 5120,512,4096 22016,512,4096 4096,512,11008 9216,2048,3072 3072,2048,3072 16384,2048,3072 3072,2048,8192 5120,2048,4096 22016,2048,4096 4096,2048,11008 > gpurun_out/r80_oos.jsonl 2> gpurun_out/r80_oos.err
