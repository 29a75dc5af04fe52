"""Bring-up check of the Llama path on the GPU vs the fp32 oracle (prints diagnostics)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import lmoracle  # noqa: E402
from paper_2604_20503_b200 import abi, engine, llama  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "tiny"
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 3
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
mode = int(sys.argv[4]) if len(sys.argv) > 4 else abi.MODE_VSD
desc = llama.PRESETS[preset]()
V = desc.target.vocab
rng = np.random.default_rng(0)
prompts = [rng.integers(0, V - 1, size=int(rng.integers(5, 40))).tolist() for _ in range(nreq)]
max_out = [int(rng.integers(8, 30)) for _ in range(nreq)]
t0 = time.time()
eng = engine.ServingEngine(desc=desc, max_batch=8, max_seq_len=256, mode=mode, default_spec_length=4,
                           debug_capture=1, max_spec_length=16, prefill_rows=2048)
print("engine create", time.time() - t0, flush=True)
t0 = time.time()
tgt = lmoracle.Model(desc.target, desc.bigram_a, desc.bigram_b)
drf = lmoracle.Model(desc.draft, desc.bigram_a, desc.bigram_b)
print("oracle create", time.time() - t0, flush=True)
for i, (p, m) in enumerate(zip(prompts, max_out)):
    eng.submit(i, p, m)
ctx = {i: list(p) for i, p in enumerate(prompts)}
worst = 0.0
acc_tot = sub_tot = 0
for s in range(steps):
    live = eng.live_requests()
    if not live:
        break
    eng.set_spec_lengths(live, [1 + (r * 3 + s) % 6 for r in live])
    if mode >= abi.MODE_VSD_AD_EE:
        eng.set_gate(abi.GatePlan(1, desc.target.layers, 1.0))
    res = eng.step()
    z, ids = eng.debug_verify_logits(0)
    dr = eng.debug_drafted()
    for li, r in enumerate(res):
        rid = r.req_id
        d = dr[li][:r.drafted].tolist()
        rows = [k for k in range(len(ids)) if ids[k][0] == rid]
        nrow = len(rows)
        ref = tgt.logits(ctx[rid] + d[:nrow - 1], len(ctx[rid]) - 1)[0]
        g = z[rows]
        rng_ = ref.max(-1) - ref.min(-1)
        err = np.abs(g - ref).max(-1) / rng_
        worst = max(worst, float(err.max()))
        # draft tokens vs oracle draft argmax
        dref = drf.logits(ctx[rid] + d[:-1], len(ctx[rid]) - 1)[0]
        dam = dref.argmax(-1)
        top2 = np.sort(dref, -1)[:, -2:]
        for j in range(len(d)):
            if dam[j] != d[j]:
                gap = (top2[j, 1] - top2[j, 0]) / (dref[j].max() - dref[j].min())
                print(f"  draft mismatch req {rid} j {j}: gpu {d[j]} oracle {dam[j]} gap {gap:.2e}")
        am = ref.argmax(-1)
        gam = g.argmax(-1)
        for j in range(nrow):
            if am[j] != gam[j]:
                t2 = np.sort(ref[j])[-2:]
                print(f"  target argmax mismatch req {rid} j {j}: gpu {gam[j]} oracle {am[j]} gap {(t2[1]-t2[0])/rng_[j]:.2e}")
        acc_tot += r.outcome.accepted_count
        sub_tot += r.outcome.submitted
        ctx[rid] += list(r.tokens[:r.committed])
    print(f"step {s}: live {len(live)} worst rel err so far {worst:.3e} accept {acc_tot}/{sub_tot}", flush=True)
for i, (p, m) in enumerate(zip(prompts, max_out)):
    got = eng.committed(i)
    ref = tgt.greedy(p, m, V - 1)
    print("req", i, "lossless" if got == ref else f"DIFF gpu {got} ref {ref}")
