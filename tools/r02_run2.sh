#!/bin/bash
# round-2 GPU call 2: GEMM chain timeline experiments (tools/layer_chain.py) + new GEMM tests
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r2_chain.jsonl; : > $O
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/r2_gemm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gemm_tests.log
run() { echo "# $*" >> $O; timeout 120 python tools/layer_chain.py "$@" >> $O 2>&1; }
run --rows 128 --trace
run --rows 128 --plan qkv=128:7,o=128:8,gu=128:2,down=128:8 --trace
run --rows 128 --plan qkv=1128:7,o=1128:8,gu=1128:2,down=1128:8 --trace
run --rows 128 --plan qkv=1128:4,o=1128:4,gu=1128:1,down=1128:4 --trace
run --rows 128 --plan qkv=20128:8,o=20128:8,gu=20128:4,down=20128:8 --trace
run --rows 128 --plan qkv=1064:4,o=1064:4,gu=1064:1,down=1064:4 --trace
run --rows 32 --trace
run --rows 256 --trace
run --rows 512
run --rows 1024
