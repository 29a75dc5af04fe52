"""Time K3 alone (graph-captured back-to-back launches) at decode/verify shapes. Every launch
reads its own KV pool (iters pools >> L2), so the pages come from HBM as in a real forward.
Args: n_req,rows,ctx[,n_q,n_kv,hd] ..."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import engine  # noqa: E402

L = engine.lib()


def run(n_req, rows, ctx, n_q=32, n_kv=4, hd=64, iters=20):
    # ATTN_BENCH_RAGGED=1: per-request contexts uniform in [ctx/4, 7 ctx/4] (mean ctx), as in a
    # continuous batch; max_ctx (grid / split decisions) is the longest
    ragged = os.environ.get("ATTN_BENCH_RAGGED") == "1"
    g = torch.Generator().manual_seed(1)
    ctxs = [int(torch.randint(max(rows, ctx // 4), ctx * 7 // 4 + 1, (1,), generator=g)) if ragged else ctx
            for _ in range(n_req)]
    max_ctx = max(ctxs)
    max_pages = (max_ctx + 63) // 64 + 1
    kvs = [torch.randn(n_req * max_pages, n_kv, 2, 64, hd, device="cuda").to(torch.bfloat16) for _ in range(iters)]
    ptab = torch.randperm(n_req * max_pages, device="cuda").to(torch.int32).view(n_req, max_pages).contiguous()
    q = torch.randn(n_req * rows, n_q, hd, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    t = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")
    first, n, pos0 = t([i * rows for i in range(n_req)]), t([rows] * n_req), t([c - rows for c in ctxs])
    scratch = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")

    def call(s, kv):
        assert L.faser_k_attention(C.c_void_p(q.data_ptr()), C.c_void_p(kv.data_ptr()), C.c_void_p(ptab.data_ptr()),
                                   max_pages, n_req, C.c_void_p(first.data_ptr()), C.c_void_p(n.data_ptr()),
                                   C.c_void_p(pos0.data_ptr()), rows, max_ctx, n_q, n_kv, hd, C.c_void_p(out.data_ptr()),
                                   C.c_void_p(scratch.data_ptr()), scratch.numel(), C.c_void_p(s)) == 0
    call(torch.cuda.current_stream().cuda_stream, kvs[0])
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for i in range(iters):
            call(torch.cuda.current_stream().cuda_stream, kvs[i])
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    kvb = sum(ctxs) * n_kv * 2 * hd * 2
    return {"n_req": n_req, "rows": rows, "ctx": ctx, "ragged": ragged, "max_ctx": max_ctx, "n_q": n_q, "n_kv": n_kv, "hd": hd, "us": round(us, 2),
            "kv_GBs": round(kvb / us / 1e3, 1)}


if __name__ == "__main__":
    for a in sys.argv[1:] or ["32,4,600", "128,4,600", "1,4,600", "32,1,600,12,12,64"]:
        print(json.dumps(run(*[int(x) for x in a.split(",")])), flush=True)
