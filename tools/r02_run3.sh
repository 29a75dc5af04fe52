#!/bin/bash
# round-2 GPU call 3: green-context lanes (FULL mode) tests + overlapped regression
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lanes_gpu.py tests/test_llama_gpu.py -q -x -rA --durations=8 > gpurun_out/r3_lanes.log 2>&1
echo "rc=$?" >> gpurun_out/r3_lanes.log
