#!/bin/bash
# round-2 GPU call 1: bench-config parity tests, full GPU suite, default bench line
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/r1_box.txt 2>&1
timeout 1200 python -m pytest tests/test_llama_bench_parity_gpu.py -x -q -rA --durations=5 > gpurun_out/r1_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/r1_parity.log
timeout 900 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r1_gpu_tests.log 2>&1
echo "suite rc=$?" >> gpurun_out/r1_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
echo "bench rc=$?" >> gpurun_out/r1_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r1_ref.json 2> gpurun_out/r1_ref.err
echo "ref rc=$?" >> gpurun_out/r1_ref.err
