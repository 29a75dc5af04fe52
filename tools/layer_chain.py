"""Verify-forward GEMM chain microbenchmark (config-3 shapes by default): L layers x
(qkv, o, gate/up, down) with distinct weights per layer (defeats L2 like a real forward),
back-to-back on one stream (PDL), graph-replayed. Prints us per layer and per GEMM class, and
with --trace a per-launch timeline from the kernel's globaltimer stamps:
  gap   = this launch's first CTA entry - previous launch's last CTA exit
  pre   = median(after griddepcontrol.wait - entry)
  fill  = median(first stage landed - after wait)
  main  = median(accumulators complete - first stage)
  red   = median(split-K reduced - accumulators complete)
  epi   = median(exit - reduced)
  span  = last exit - first entry
Usage: python tools/layer_chain.py --rows 128 [--plan qkv=CODE:SPLITS,...] [--trace]
CODE = 10000*mc + 1000*depth + bn (0 = the engine planner)."""
import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import engine  # noqa: E402

L = engine.lib()
SHAPES = {"cfg3": {"qkv": (2560, 2048), "o": (2048, 2048), "gu": (11264, 2048), "down": (2048, 5632)},
          "cfg4": {"qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336)},
          # config-3 draft (llama-68m shape) and its LM head (the draft's other GEMM per step)
          "draft": {"qkv": (2304, 768), "o": (768, 768), "gu": (6144, 768), "down": (768, 3072)},
          "draft_lm": {"lm": (32000, 768)}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=128)
    ap.add_argument("--layers", type=int, default=22)
    ap.add_argument("--model", default="cfg3")
    ap.add_argument("--plan", default="")
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    shapes = SHAPES[a.model]
    plan = {k: (0, 0) for k in shapes}
    for item in filter(None, a.plan.split(",")):
        name, v = item.split("=")
        c, s = v.split(":")
        plan[name] = (int(c), int(s))
    T = a.rows
    ws = {n: [(torch.randn(no, k, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(a.layers)]
          for n, (no, k) in shapes.items()}
    xs = {n: torch.randn(T, k, device="cuda").to(torch.bfloat16) for n, (no, k) in shapes.items()}
    outs = {n: torch.empty(T, no, device="cuda") for n, (no, k) in shapes.items()}
    order = list(shapes)
    plans = {}
    for n, (no, k) in shapes.items():
        o4 = (C.c_int32 * 4)()
        L.faser_k_gemm_plan(no, T, k, o4)
        plans[n] = list(o4)

    def grid(n):
        no, k = shapes[n]
        code, sp = plan[n]
        bn = code % 1000 or plans[n][0]
        mc = code // 10000 or plans[n][2]
        kb = k // 64
        s1 = min(sp or plans[n][1], 8)
        kps = (kb + s1 - 1) // s1
        z = (kb + kps - 1) // kps
        return ((no // 128 + mc - 1) // mc) * ((T + bn - 1) // bn) * z

    traces = []
    if a.trace:
        for l in range(a.layers):
            for n in order:
                traces.append((l, n, torch.zeros(grid(n) * 8, dtype=torch.int64, device="cuda")))

    def launch(stream, with_trace):
        ti = 0
        for l in range(a.layers):
            for n in order:
                no, k = shapes[n]
                code, sp = plan[n]
                tr = C.c_void_p(traces[ti][2].data_ptr()) if with_trace else None
                ti += 1
                rc = L.faser_k_gemm_bf16_trace(C.c_void_p(ws[n][l].data_ptr()), C.c_void_p(xs[n].data_ptr()),
                                               C.c_void_p(outs[n].data_ptr()), no, T, k, code, sp,
                                               C.c_void_p(stream), tr)
                assert rc == 0, rc

    s = torch.cuda.current_stream().cuda_stream
    launch(s, False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        launch(torch.cuda.current_stream().cuda_stream, False)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(a.reps):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    wbytes = sum(2 * no * k for no, k in shapes.values())
    res = {"rows": T, "model": a.model, "plans": {n: plans[n] if plan[n] == (0, 0) else list(plan[n]) for n in order},
           "us_per_layer": round(best / a.layers, 2), "GBs": round(wbytes / (best / a.layers) / 1e3, 1),
           "frac_hbm": round(wbytes / (best / a.layers) / 1e3 / 6500.3, 3)}
    # per-class timing: each class alone (same chain minus the others)
    for n in order:
        keep = order
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            cs = torch.cuda.current_stream().cuda_stream
            for l in range(a.layers):
                no, k = shapes[n]
                code, sp = plan[n]
                L.faser_k_gemm_bf16_trace(C.c_void_p(ws[n][l].data_ptr()), C.c_void_p(xs[n].data_ptr()),
                                          C.c_void_p(outs[n].data_ptr()), no, T, k, code, sp, C.c_void_p(cs), None)
        g2.replay()
        torch.cuda.synchronize()
        bb = 1e9
        for _ in range(a.reps):
            e0.record()
            g2.replay()
            e1.record()
            torch.cuda.synchronize()
            bb = min(bb, e0.elapsed_time(e1) * 1e3)
        no, k = shapes[n]
        res[f"{n}_alone_us"] = round(bb / a.layers, 2)
        res[f"{n}_alone_GBs"] = round(2 * no * k / (bb / a.layers) / 1e3, 1)
        del keep
    print(json.dumps(res), flush=True)
    if a.trace:
        launch(s, True)
        torch.cuda.synchronize()
        prev_end = None
        rows = []
        for (l, n, t) in traces:
            v = t.view(-1, 8).cpu().double()
            ent, wt, first, acc, red, ex, syn = (v[:, i] for i in range(7))
            syn = torch.where(syn > 0, syn, acc)
            ok = ex > 0
            med = lambda x: float(x[ok].median()) / 1e3  # noqa: E731
            r = {"layer": l, "gemm": n, "ctas": int(v.shape[0]),
                 "gap_us": None if prev_end is None else round((float(ent[ok].min()) - prev_end) / 1e3, 2),
                 "pre_us": round(med(wt - ent), 2), "fill_us": round(med(first - wt), 2),
                 "main_us": round(med(acc - first), 2), "sync_us": round(med(syn - acc), 2), "red_us": round(med(red - syn), 2),
                 "epi_us": round(med(ex - red), 2),
                 "span_us": round((float(ex[ok].max()) - float(ent[ok].min())) / 1e3, 2),
                 "entry_spread_us": round((float(ent[ok].max()) - float(ent[ok].min())) / 1e3, 2)}
            prev_end = float(ex[ok].max())
            rows.append(r)
        for r in rows[len(order):len(order) * 3]:  # layers 1-2 (steady state)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
