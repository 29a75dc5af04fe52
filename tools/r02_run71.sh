#!/bin/bash
# round-2 GPU call 71: toy admission fused into the round kernel
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_toy_gpu.py -q -x > gpurun_out/r71_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r71_tests.log
grep -q "rc=0" gpurun_out/r71_tests.log || exit 3
FASER_TOY_PROF=1 timeout 300 python bench.py --workload toy --steps 200 --warmup 20 > gpurun_out/r71_toy.json 2> gpurun_out/r71_toy.err
