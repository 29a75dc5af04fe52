#!/bin/bash
# round-2 GPU call 7: split-K reduce breakdown (cluster wait vs DSMEM reduce)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r7_chain.jsonl; : > $O
run() { echo "# $*" >> $O; timeout 120 python tools/layer_chain.py "$@" >> $O 2>&1; }
run --rows 128 --trace
run --rows 128 --plan qkv=1128:7,o=1128:8,gu=1064:1,down=1128:8 --trace
run --rows 128 --plan qkv=1064:4,o=1064:4,gu=1064:1,down=1064:4 --trace
