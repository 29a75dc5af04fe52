#!/bin/bash
# round-2 GPU call 53: attention fixed cost vs per-page cost (ctx sweep), both kernels, + empty-kernel floor
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
O=gpurun_out/r53_attn_ctx.txt; : > $O
for cfg in "FASER_ATTN_TC=1" "FASER_ATTN_TC=0"; do
  echo "== $cfg" >> $O
  env $cfg timeout 120 python tools/attn_bench.py 32,4,8 32,4,64 32,4,128 32,4,256 32,4,512 32,4,1024 32,4,2048 8,4,64 8,4,600 1,4,64 1,4,600 >> $O 2>&1
done
python - >> $O 2>&1 <<'PY'
import torch
x = torch.zeros(1, device="cuda")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(20): x.add_(1)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print("empty-ish kernel per launch in graph (us):", e0.elapsed_time(e1) * 1e3 / 20)
PY
