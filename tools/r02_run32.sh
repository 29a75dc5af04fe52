#!/bin/bash
# round-2 GPU call 32: in-stream class costs in the bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline > gpurun_out/r32_bench.json 2> gpurun_out/r32_bench.err; echo "rc=$?" >> gpurun_out/r32_bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --batch 128 > gpurun_out/r32_bench128.json 2>> gpurun_out/r32_bench.err
