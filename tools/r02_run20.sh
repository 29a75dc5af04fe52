#!/bin/bash
# round-2 GPU call 20: default bench line at HEAD (kernel classes timed with the prefill lane off),
# 20-step driver-style line, config-4 line, full GPU suite
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/r20_bench.json 2> gpurun_out/r20_bench.err; echo "bench rc=$?" >> gpurun_out/r20_bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r20_bench_s20.json 2>> gpurun_out/r20_bench.err
timeout 900 python bench.py --workload cfg4 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline > gpurun_out/r20_cfg4.json 2>> gpurun_out/r20_bench.err
timeout 900 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r20_gpu_tests.log 2>&1; echo "suite rc=$?" >> gpurun_out/r20_gpu_tests.log
