#!/bin/bash
# round-2 GPU call 6: GEMM chain plan experiments at 128 rows (co-resident shallow grids <= 148 CTAs)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r6_chain.jsonl; : > $O
run() { echo "# $*" >> $O; timeout 120 python tools/layer_chain.py "$@" >> $O 2>&1; }
run --rows 128
run --rows 128 --plan qkv=1128:7,o=1128:8,gu=1128:1,down=1128:8 --trace
run --rows 128 --plan qkv=1128:7,o=1128:8,gu=1064:1,down=1128:8 --trace
run --rows 128 --plan qkv=1128:7,o=1128:8,gu=20128:2,down=1128:8 --trace
run --rows 128 --plan qkv=1064:4,o=1064:4,gu=1064:1,down=1064:4 --trace
run --rows 128 --plan qkv=2128:7,o=2128:8,gu=2128:1,down=2128:8 --trace
run --rows 128 --plan qkv=1032:2,o=1032:2,gu=1064:1,down=1064:4
run --rows 128 --plan qkv=1128:4,o=1128:4,gu=1128:1,down=1128:4
