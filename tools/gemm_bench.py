"""Time the tcgen05 GEMM alone at verify/draft shapes (CUDA events, L2 flushed between
iterations) and print achieved GB/s (weights) and TFLOP/s."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import engine  # noqa: E402

L = engine.lib()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
shapes = [(2560, 20, 2048), (2048, 160, 2048), (11264, 160, 2048), (2048, 160, 5632),
          (32000, 160, 2048), (11264, 32, 2048), (11264, 1280, 2048), (2048, 1280, 5632),
          (14336 * 2, 160, 4096), (4096, 160, 14336), (6144, 32, 768), (32000, 32, 768)]
for n, t, k in [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]] or shapes:
    w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    x = torch.randn(t, k, device="cuda").to(torch.bfloat16)
    out = torch.empty(t, n, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ts = []
    for i in range(12):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert L.faser_k_gemm_bf16(C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()),
                                   C.c_void_p(out.data_ptr()), n, t, k, 0, C.c_void_p(s)) == 0
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(json.dumps({"n": n, "t": t, "k": k, "us": round(ms * 1e3, 2),
                      "weight_GBs": round(2 * n * k / ms / 1e6, 1),
                      "TFLOPs": round(2 * n * k * t / ms / 1e9, 1)}))
