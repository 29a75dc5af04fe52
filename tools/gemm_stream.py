"""Steady-state streaming rate of the tcgen05 GEMM: back-to-back launches cycling over enough
weight copies to defeat L2 (like consecutive layers of a forward). Prints us/launch and GB/s."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import engine  # noqa: E402

L = engine.lib()


def run(n, t, k, bn=0, splits=0, iters=60):
    copies = max(2, (256 << 20) // (n * k * 2) + 1)
    ws = [(torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(copies)]
    x = torch.randn(t, k, device="cuda").to(torch.bfloat16)
    out = torch.empty(t, n, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for i in range(copies):
        assert L.faser_k_gemm_bf16_plan(C.c_void_p(ws[i].data_ptr()), C.c_void_p(x.data_ptr()),
                                        C.c_void_p(out.data_ptr()), n, t, k, bn, splits, C.c_void_p(s)) == 0
    # capture the launch sequence in a CUDA graph so host launch overhead is excluded
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        cs = torch.cuda.current_stream().cuda_stream
        for i in range(iters):
            L.faser_k_gemm_bf16_plan(C.c_void_p(ws[i % copies].data_ptr()), C.c_void_p(x.data_ptr()),
                                     C.c_void_p(out.data_ptr()), n, t, k, bn, splits, C.c_void_p(cs))
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    return {"n": n, "t": t, "k": k, "bn": bn, "splits": splits, "us": round(us, 2),
            "GBs": round(2 * n * k / us / 1e3, 1), "TFLOPs": round(2 * n * k * t / us / 1e6, 1)}


if __name__ == "__main__":
    cases = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
    for c in cases:
        print(json.dumps(run(*c)), flush=True)
