"""Rank of the drafted token in the gated-layer logits, split by whether the final verify
accepted it — how predictive token-wise early exit can be on this model."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import abi, engine, llama  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
layers = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "6,11,16").split(",")]
desc = llama.PRESETS[preset]()
L = desc.target.layers
eng = engine.ServingEngine(desc=desc, max_batch=16, max_seq_len=600, mode=abi.MODE_VSD_AD_EE,
                           default_spec_length=6, debug_capture=1, max_spec_length=16, prefill_rows=4096,
                           exit_policy=abi.ExitPolicy(1, 1000000, 1000000))
rng = np.random.default_rng(0)
for i in range(16):
    eng.submit(i, rng.integers(0, desc.target.vocab - 1, size=200).tolist(), 60)
ranks = {l: {"acc": [], "rej": []} for l in layers}
for step in range(12):
    if not eng.live_requests():
        break
    eng.set_gate(abi.GatePlan(min(layers), max(layers) + 1, 1.0))
    res = eng.step()
    dr = eng.debug_drafted()
    zf, idf = eng.debug_verify_logits(0)
    for li, r in enumerate(res):
        d = dr[li][:r.drafted]
        frow = {int(idf[q][1]): q for q in range(len(idf)) if idf[q][0] == r.req_id}
        truth = [int(np.argmax(zf[frow[j]])) for j in range(len(d))]
        first_bad = next((j for j in range(len(d)) if truth[j] != d[j]), len(d))
        for l in layers:
            z, ids = eng.debug_verify_logits(l)
            rowof = {int(ids[q][1]): q for q in range(len(ids)) if ids[q][0] == r.req_id}
            for j in range(min(first_bad + 1, len(d))):
                zz = z[rowof[j]]
                rank = int((zz > zz[d[j]]).sum())
                (ranks[l]["acc"] if j < first_bad else ranks[l]["rej"]).append(rank)
for l in layers:
    a, rj = np.array(ranks[l]["acc"]), np.array(ranks[l]["rej"])
    q = lambda x, p: float(np.percentile(x, p)) if len(x) else -1
    print(f"layer {l}/{L}: accepted n={len(a)} rank p50 {q(a,50)} p90 {q(a,90)} p99 {q(a,99)} | "
          f"rejected n={len(rj)} rank p10 {q(rj,10)} p50 {q(rj,50)} | "
          + " ".join(f"K={K}: prune_rej {np.mean(rj >= K):.2f} false_prune {np.mean(a >= K):.3f}" for K in (1, 2, 5, 10, 50)))
