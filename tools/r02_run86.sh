#!/bin/bash
# round-2 GPU call 86: ncu --set full of one config-3 B=32 serving step at HEAD: verify layer-0 GEMMs + attention (traffic for bench.py roofline)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
PROFILE_ONE_STEP=1 PERF_STEPS=3 timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:gemm_kernel --launch-skip 36 -c 4 -o gpurun_out/r86_gemm python tools/llama_perf.py cfg3 32 4 > gpurun_out/r86_gemm.log 2>&1
PROFILE_ONE_STEP=1 PERF_STEPS=3 timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:attn --launch-skip 8 -c 1 -o gpurun_out/r86_attn python tools/llama_perf.py cfg3 32 4 > gpurun_out/r86_attn.log 2>&1
