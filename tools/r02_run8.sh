#!/bin/bash
# round-2 GPU call 8: L2 prefetch of the CTA weight slice before the PDL wait (FASER_L2_PF=1)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r8_chain.jsonl; : > $O
run() { echo "# $*" >> $O; timeout 120 python tools/layer_chain.py "$@" >> $O 2>&1; }
for pf in 0 1; do
export FASER_L2_PF=$pf
echo "## L2PF=$pf" >> $O
run --rows 128 --trace
run --rows 128 --plan qkv=1128:7,o=1128:8,gu=1128:1,down=1128:8 --trace
run --rows 128 --plan qkv=1064:4,o=1064:4,gu=1128:1,down=1064:4 --trace
run --rows 32
run --rows 256
done
