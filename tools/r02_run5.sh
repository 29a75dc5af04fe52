#!/bin/bash
# round-2 GPU call 5 (session 3): full GPU suite at HEAD, GEMM chain timelines, default bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
(nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/r5_box.txt 2>&1
O=gpurun_out/r5_chain.jsonl; : > $O
run() { echo "# $*" >> $O; timeout 120 python tools/layer_chain.py "$@" >> $O 2>&1; }
run --rows 128 --trace
run --rows 32 --trace
run --rows 512 --trace
timeout 900 python bench.py --steps 20 --warmup 5 --no-sweep > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err
echo "bench rc=$?" >> gpurun_out/r5_bench.err
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r5_gpu_tests.log 2>&1
echo "suite rc=$?" >> gpurun_out/r5_gpu_tests.log
