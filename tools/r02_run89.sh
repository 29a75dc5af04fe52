#!/bin/bash
# round-2 GPU call 89: online-profiler GPU test, run-bracketed class timing in the bench, ablate with online refits
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_trace_gpu.py tests/test_llama_gpu.py -q -x > gpurun_out/r89_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r89_tests.txt
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r89_bench_s20.json 2> gpurun_out/r89_bench_s20.err
timeout 900 python tools/ablate.py --workload cfg3 --seconds 4 --rate 120 --batch 64 --modes VSD_AD --refresh-steps 32 --out gpurun_out/r89_ablate_refresh > gpurun_out/r89_ablate.txt 2>&1
timeout 900 python tools/ablate.py --workload cfg3 --seconds 4 --rate 120 --batch 64 --modes VSD_AD --out gpurun_out/r89_ablate_norefresh >> gpurun_out/r89_ablate.txt 2>&1
