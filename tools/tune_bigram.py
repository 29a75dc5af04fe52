"""Acceptance rate of the Llama preset vs the target bigram strength (greedy, fixed k=4)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import abi, engine, llama  # noqa: E402

preset = sys.argv[1]
betas = [float(b) for b in sys.argv[2].split(",")]
hard = float(sys.argv[3]) if len(sys.argv) > 3 else None
for beta in betas:
    desc = llama.PRESETS[preset](target_bigram=beta, hard=hard)
    V = desc.target.vocab
    rng = np.random.default_rng(1)
    eng = engine.ServingEngine(desc=desc, max_batch=16, max_seq_len=512, mode=abi.MODE_VSD,
                               default_spec_length=4, max_spec_length=16, prefill_rows=4096)
    for i in range(16):
        eng.submit(i, rng.integers(0, V - 1, size=128).tolist(), 64)
    acc = sub = steps = 0
    while eng.live_requests():
        for r in eng.step():
            acc += r.outcome.accepted_count
            sub += r.outcome.submitted
        steps += 1
    print(f"{preset} target_bigram {beta}: accept {acc}/{sub} = {acc / sub:.3f} steps {steps}", flush=True)
    eng.close()
