#!/bin/bash
# round-2 GPU call 9: ingest-minimising plans at 128 rows (BN = all rows, MC weight tiles per rows tile)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r9_chain.jsonl; : > $O
run() { echo "# $*" >> $O; timeout 120 python tools/layer_chain.py "$@" >> $O 2>&1; }
run --rows 128
run --rows 128 --plan qkv=2128:4,o=2128:8,gu=2128:1,down=2128:8
run --rows 128 --plan qkv=2128:7,o=20128:8,gu=20128:1,down=20128:8
run --rows 128 --plan qkv=20128:4,o=40128:8,gu=20128:2,down=40128:8
run --rows 128 --plan qkv=20128:8,o=20128:4,gu=40128:2,down=20128:4
run --rows 128 --plan qkv=40128:8,o=2128:4,gu=40128:4,down=2128:4
run --rows 128 --plan qkv=1128:4,o=1128:8,gu=40128:6,down=1128:8
run --rows 128 --plan qkv=20064:8,o=20064:8,gu=20064:2,down=20064:8
run --rows 128 --plan qkv=40064:8,o=40064:8,gu=40064:4,down=40064:8
run --rows 128 --plan qkv=20032:8,o=20032:8,gu=20032:2,down=20032:8
