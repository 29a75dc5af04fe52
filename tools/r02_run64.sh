#!/bin/bash
# round-2 GPU call 64: host turnaround per step (Python loop and engine host time) at B=32
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
BENCH_HOST_PROF=1 FASER_PF_DEBUG=1 timeout 600 python bench.py --steps 40 --warmup 6 --no-sweep --no-cpu-baseline > gpurun_out/r64_bench.json 2> gpurun_out/r64_host.txt
