#!/bin/bash
# round-2 GPU call 57: draft GEMM split-K sweep at 32 rows (llama-68m shapes)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r57_draft_split.jsonl; : > $O
for sp in 1 2 3 4 6; do
  timeout 120 python tools/layer_chain.py --model draft --rows 32 --layers 2 --plan qkv=0:$sp,o=0:$sp,gu=0:$sp,down=0:$sp >> $O 2>&1
done
for sp in 8 12; do
  timeout 120 python tools/layer_chain.py --model draft --rows 32 --layers 2 --plan down=0:$sp,o=0:$sp,qkv=0:$sp >> $O 2>&1
done
for mc in 1 2; do for sp in 1 2; do
  timeout 120 python tools/layer_chain.py --model draft --rows 32 --layers 2 --plan qkv=${mc}0032:$sp,o=${mc}0032:$sp,gu=${mc}0032:$sp,down=${mc}0032:$sp >> $O 2>&1
done; done
