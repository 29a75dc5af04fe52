#!/bin/bash
# round-2 GPU call 13: ncu of prefill-size GEMMs (576 rows)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/gemm_bench.py 2560,576,2048 11264,576,2048 2048,576,5632 2048,576,2048 > gpurun_out/r13_gemm576.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/r13_qkv576 python tools/gemm_bench.py 2560,576,2048 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/r13_gu576 python tools/gemm_bench.py 11264,576,2048 > /dev/null 2>&1
