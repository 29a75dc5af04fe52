#!/bin/bash
# round-2 GPU call 101: config 5 at full size, TP=4 shards (padded vocab-parallel LM head) on one B200 (in-process group) vs the unsharded engine
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
(while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/r101_mem.txt; sleep 5; done) &
MON=$!
timeout 600 python -m pytest tests/test_tp_gpu.py tests/test_sampling_gpu.py -q -x > gpurun_out/r101_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r101_tests.txt
timeout 1500 python tools/cfg5_tp_onegpu.py 4 > gpurun_out/r101_cfg5_tp8.json 2> gpurun_out/r101_cfg5_tp8.err; echo "rc=$?" >> gpurun_out/r101_cfg5_tp8.err
kill $MON
