"""Full graph-timed sweep of every launch plan the GEMM kernel set instantiates, for fitting and
validating the sweep-driven planner (tc_gemm.cu gemm_plan_table, tools/gen_plan_table.py). For each (n_out, rows, k) every
(bn, mc, depth) candidate x K split is timed as back-to-back launches cycling over weight copies
that defeat L2 (like consecutive layers). One JSON line per timed plan.
Usage: python tools/plan_fit_sweep.py N,T,K [N,T,K ...]"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import engine  # noqa: E402

L = engine.lib()
# (bn, mc, deep) — the instantiated set (tc_gemm.cu gemm_fused / kPlanCands)
CANDS = [(32, 1, 1), (32, 1, 0), (64, 1, 1), (64, 1, 0), (128, 1, 1), (128, 1, 0), (256, 1, 1), (256, 1, 0),
         (32, 2, 1), (64, 2, 1), (128, 2, 1), (256, 2, 1), (32, 4, 1), (64, 4, 1), (128, 4, 1)]
SPLITS = (1, 2, 3, 4, 6, 8)


def sweep(n, t, k, iters=20):
    copies = max(2, (256 << 20) // (n * k * 2) + 1)
    ws = [(torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(copies)]
    x = torch.randn(t, k, device="cuda").to(torch.bfloat16)
    out = torch.empty(t, n, device="cuda")
    kb = k // 64
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for bn, mc, deep in CANDS:
        if mc > 1 and n // 128 < mc:
            continue
        if bn > 32 and bn // 2 >= t:
            continue
        code = mc * 10000 + (2 if deep else 1) * 1000 + bn
        for sp in SPLITS:
            kps = (kb + sp - 1) // sp
            if sp > 1 and (kps < 4 or (kb + kps - 1) // kps != sp):
                continue

            def launch(i, s):
                return L.faser_k_gemm_bf16_plan(C.c_void_p(ws[i % copies].data_ptr()), C.c_void_p(x.data_ptr()),
                                                C.c_void_p(out.data_ptr()), n, t, k, code, sp, C.c_void_p(s))
            if launch(0, torch.cuda.current_stream().cuda_stream) != 0:
                continue
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                cs = torch.cuda.current_stream().cuda_stream
                for i in range(iters):
                    launch(i, cs)
            g.replay()
            torch.cuda.synchronize()
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / iters
            print(json.dumps({"n": n, "t": t, "k": k, "bn": bn, "mc": mc, "deep": deep, "splits": sp,
                              "us": round(us, 2)}), flush=True)
            del g


if __name__ == "__main__":
    for a in sys.argv[1:]:
        sweep(*[int(v) for v in a.split(",")])
