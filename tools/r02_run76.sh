#!/bin/bash
# round-2 GPU call 76: prefill-size GEMM chain (rows 576 / 2048 / 8192): TFLOP/s per class; ncu of gate/up at 4096 rows
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r76_prefill_chain.jsonl; : > $O
for r in 576 2048 4096 8192; do timeout 300 python tools/layer_chain.py --rows $r --layers 4 --reps 3 >> $O 2>&1; done
timeout 300 ncu --set full --clock-control none -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/r76_gu python tools/layer_chain.py --rows 4096 --layers 1 --reps 1 > gpurun_out/r76_ncu.log 2>&1
