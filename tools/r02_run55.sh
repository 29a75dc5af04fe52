#!/bin/bash
# round-2 GPU call 55: draft GEMM chain (llama-68m shapes, 32 rows): per-GEMM timeline, L2-warm (2 layers) vs cold (22)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r55_draft_chain.jsonl; : > $O
for rows in 32 40; do
  timeout 120 python tools/layer_chain.py --model draft --rows $rows --layers 2 --trace >> $O 2>&1
  timeout 120 python tools/layer_chain.py --model draft --rows $rows --layers 22 >> $O 2>&1
  timeout 120 python tools/layer_chain.py --model draft_lm --rows $rows --layers 2 --trace >> $O 2>&1
  timeout 120 python tools/layer_chain.py --model draft_lm --rows $rows --layers 8 >> $O 2>&1
done
