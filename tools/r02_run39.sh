#!/bin/bash
# round-2 GPU call 39: native serving loop for the toy path; prefill lane in EE mode
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_toy_gpu.py tests/test_llama_gpu.py -q -x -k "native or prefill_lane" > gpurun_out/r39_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r39_tests.log
timeout 300 python bench.py --workload toy --steps 200 --warmup 20 > gpurun_out/r39_toy.json 2> gpurun_out/r39_toy.err; echo "rc=$?" >> gpurun_out/r39_toy.err
timeout 300 python bench.py --workload toy --impl reference --steps 200 --warmup 20 > gpurun_out/r39_toy_ref.json 2>> gpurun_out/r39_toy.err
