#!/bin/bash
# round-2 GPU call 90: coupled Gumbel-max sampling acceptance — tests (+ the GEMM / Llama suites the epilogue touches), a sampling bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sampling_gpu.py -q -x > gpurun_out/r90_sampling.txt 2>&1; echo "rc=$?" >> gpurun_out/r90_sampling.txt
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_llama_gpu.py tests/test_tp_gpu.py -q -x > gpurun_out/r90_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r90_tests.txt
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-sweep --temperature 1.0 > gpurun_out/r90_bench_t1.json 2> gpurun_out/r90_bench_t1.err
