#!/bin/bash
# round-2 GPU call 78: draft GEMM chain, shallow (2 CTAs/SM) vs deep (1 CTA/SM) pipelines: PDL overlap gaps
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r78_draft_depth.jsonl; : > $O
for d in 1 2; do
  echo "{\"depth\": $d}" >> $O
  timeout 120 python tools/layer_chain.py --model draft --rows 32 --layers 2 --trace --plan qkv=${d}032:3,o=${d}032:3,gu=${d}032:1,down=${d}032:8 >> $O 2>&1
  timeout 120 python tools/layer_chain.py --model draft --rows 32 --layers 22 --plan qkv=${d}032:3,o=${d}032:3,gu=${d}032:1,down=${d}032:8 >> $O 2>&1
done
